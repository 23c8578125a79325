mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider -k "ranks or streamed or distributed or serialised" > gpurun_out/pytest_ranks.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_ranks.log
python bench.py --steps 3 --warmup 3 --no-steps --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['value'],d['kernel_ms'],d['e2e'])"
timeout 900 python tools/emulate_scaling.py > gpurun_out/emulate.log 2>&1; echo emu_rc=$?
tail -6 gpurun_out/emulate.log
