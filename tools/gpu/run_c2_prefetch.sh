# C2 kernel time vs the ahead-of-time claim threshold (TINV_PREFETCH_MIN; 0 = off)
mkdir -p gpurun_out
for pf in 0 1 2 4 8 16 0; do
  r=$(TINV_PREFETCH_MIN=$pf timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-steps --no-load 2>/dev/null | tail -1)
  echo "pf=$pf $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"
done
for pf in 0 2 8; do
  r=$(TINV_PREFETCH_MIN=$pf timeout 300 python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu --no-steps --no-load 2>/dev/null | tail -1)
  echo "c3 pf=$pf $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')"
done
