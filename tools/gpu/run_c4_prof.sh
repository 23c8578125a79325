mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "fused" -p no:cacheprovider > gpurun_out/c4_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/c4_tests.log
for slots in 3 4; do
TINV_BPIPE_SLOTS=$slots timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4_pipe$slots.json 2> gpurun_out/bench_c4_pipe$slots.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c4_pipe$slots.json'));print('slots $slots', d['value'], d['kernel_ms'], d['roofline']['frac'])"
TINV_BPIPE_SLOTS=$slots TINV_BPIPE_PROF=1 timeout 300 python bench.py --workload c4 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep "bpipe\]" | tail -2
done
