# A/B of two library builds (TINV_LIB) on C1 and C2, interleaved
for rep in 1 2 3; do
  for lib in tools/micro/libtileinv_old.so paper_1002_4057_b200/libtileinv_b200.so; do
    for w in c1 c2; do
      r=$(TINV_LIB=$lib timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu --no-steps --no-load 2>/dev/null | tail -1)
      echo "$lib $w $(echo "$r" | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d.get("kernel_ms",0),3))')"
    done
  done
done
