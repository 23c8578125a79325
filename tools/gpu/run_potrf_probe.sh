mkdir -p gpurun_out
timeout 120 python tools/potrf_probe.py 256 2
timeout 120 python tools/potrf_probe.py 256 4
TINV_PHASE_PROFILE=1 timeout 120 python tools/potrf_probe.py 256 2 2>&1 | grep -E "phase\]" | tail -3
timeout 120 python tools/potrf_probe.py 128 2
