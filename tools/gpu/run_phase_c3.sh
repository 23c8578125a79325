mkdir -p gpurun_out
TINV_PHASE_PROFILE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load 2>&1 | grep "phase\]" | tail -3
