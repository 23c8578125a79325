mkdir -p gpurun_out
TINV_PHASE_PROFILE=1 timeout 300 python tools/potrf_probe.py 256 2 2>&1 | tail -12
TINV_PHASE_PROFILE=1 timeout 300 python tools/potrf_probe.py 128 2 2>&1 | tail -12
