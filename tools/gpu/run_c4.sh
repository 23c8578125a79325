# C4 engines: parity tests of the fused batched path, then the bench line (pipelined engine vs one-CTA-per-matrix)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "fused" -p no:cacheprovider > gpurun_out/c4_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/c4_tests.log
timeout 300 python -m pytest tests/test_gpu_full.py -q -x -k "c4" -p no:cacheprovider > gpurun_out/c4_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/c4_full.log
for slots in 2 3 4; do
TINV_BPIPE_SLOTS=$slots timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4_pipe$slots.json 2> gpurun_out/bench_c4_pipe$slots.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c4_pipe$slots.json'));print('slots $slots', d['value'], d['kernel_ms'], d['roofline']['frac'])"
TINV_BPIPE_SLOTS=$slots TINV_BPIPE_PROF=1 timeout 300 python bench.py --workload c4 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep "bpipe\]" | tail -1
done
