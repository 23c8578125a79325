# block Cholesky change: GPU parity tests, step-1 chain latencies, C1/C2 bench, C2 phase/idle profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/potrf_probe.py 256 2 2>&1 | tail -5
timeout 300 python tools/potrf_probe.py 128 2 2>&1 | tail -5
for w in c1 c2; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steps --no-load 2>/dev/null | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["ms_per_step"], d["value"])'
done
TINV_PHASE_PROFILE=1 timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-steps --no-load 2>&1 | grep "phase\]" | tail -4
