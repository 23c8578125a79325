# full GPU suite, then the reference arm and the default bench (driver-style)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -s -p no:cacheprovider -rs --durations=12 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "normwise|passed|failed|FAILED|Error" gpurun_out/pytest.log | head -30
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref_rc=$?
tail -c 1500 gpurun_out/ref.json
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.json
