mkdir -p gpurun_out
TINV_BPIPE_SLOTS=${SLOTS:-3} TINV_BPIPE_PROF=1 timeout 300 python bench.py --workload c4 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | grep "bpipe\]" | tail -3
TINV_BPIPE_SLOTS=${SLOTS:-3} timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4', d['value'], d['kernel_ms'], d['roofline']['frac'])"
