mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "fused" -p no:cacheprovider > gpurun_out/c4_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c4_tests.log
for sl in ${SLOTS:-3}; do
TINV_BPIPE_SLOTS=$sl TINV_BPIPE_PROF=1 timeout 300 python bench.py --workload c4 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep "bpipe\]" | tail -3
TINV_BPIPE_SLOTS=$sl timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4 slots $sl', d['value'], d['kernel_ms'], d['roofline']['frac'])"
done
