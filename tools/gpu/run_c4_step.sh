# C4 iteration: fused parity tests, then the bench kernel time twice
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "fused" -p no:cacheprovider > gpurun_out/c4_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/c4_tests.log
for rep in 1 2; do
TINV_BSMALL_PROF=$PROF timeout 300 python bench.py --workload c4 --fused-engine cta --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4_cta.json 2>gpurun_out/bench_c4_cta.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c4_cta.json'));print('c4 cta', d['value'], d['kernel_ms'], d['roofline']['frac'])"
done
TINV_BSMALL_PROF=1 python tools/bsmall_probe.py 8192 256 2>&1 | grep -E "cycles per matrix" | tail -1
