mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gpu_tests.log
for w in c2 c1; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/final_$w.json 2> gpurun_out/final_$w.err; echo ${w}_rc=$?
python -c "import json;d=json.load(open('gpurun_out/final_$w.json'));e=d.get('e2e') or {};print('$w', round(d['value']), round(d['kernel_ms'],3), round(d['roofline']['frac'],4), 'e2e', round(e.get('value') or 0))"
done
TINV_READY_PROFILE=1 timeout 500 python tools/critpath.py 8192 256 out 2>&1 | head -14
