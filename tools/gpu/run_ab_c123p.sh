bash tools/gpu/run_ab_c123.sh
TINV_PHASE_PROFILE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load 2>&1 | grep "phase\] per item"
TINV_PHASE_PROFILE=1 timeout 600 python bench.py --workload c2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load 2>&1 | grep "phase\] per item"
python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider -k "not multi_process and not multi_rank" 2>&1 | tail -1
