# C2 per-item phase profile (TINV_PHASE_PROFILE=1) + dispatch split (TINV_READY_PROFILE=1)
mkdir -p gpurun_out
TINV_PHASE_PROFILE=1 timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/phase_c2.log 2>&1
grep "phase\]" gpurun_out/phase_c2.log | tail -3
tail -1 gpurun_out/phase_c2.log | cut -c1-300
