mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_cli.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests.log
timeout 120 python tools/potrf_probe.py 256 4 | head -8
timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/c2.json 2> gpurun_out/c2.err; echo c2 rc=$?
python -c "import json;d=json.load(open('gpurun_out/c2.json'));print('c2', round(d['value']), round(d['kernel_ms'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), d['residual'])"
timeout 300 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu --no-load > gpurun_out/c1.json 2> gpurun_out/c1.err; echo c1 rc=$?
python -c "import json;d=json.load(open('gpurun_out/c1.json'));print('c1', round(d['value']), round(d['kernel_ms'],3))"
