mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
for w in c3 c2; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; echo ${w}_rc=$?
python -c "import json;d=json.load(open('gpurun_out/b_$w.json'));print('$w', round(d['value']), round(d['kernel_ms'],2), round(d['roofline']['frac'],4))"
done
TINV_PHASE_PROFILE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load 2>&1 | grep "phase\]" | tail -3
