mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py tests/test_gpu_full.py -q -x -k "fused or c4" -p no:cacheprovider > gpurun_out/c4_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/c4_tests.log
for eng in pipe cta; do
timeout 300 python bench.py --workload c4 --fused-engine $eng --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4_$eng.json 2>gpurun_out/bench_c4_$eng.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c4_$eng.json'));print('c4 $eng', d['value'], d['kernel_ms'], d['roofline']['frac'])"
done
TINV_BPIPE_PROF=1 timeout 300 python bench.py --workload c4 --fused-engine pipe --steps 2 --warmup 1 --no-e2e --no-cpu 2> gpurun_out/bpipe_prof.log >/dev/null; grep "bpipe\]" gpurun_out/bpipe_prof.log | tail -4
