mkdir -p gpurun_out/ktrim
for nb in 200 136 72; do
for v in 1 0; do
TINV_NO_KTRIM=$v python bench.py --n $((nb*32)) --nb $nb --steps 5 --warmup 3 --no-e2e --no-cpu --no-load > gpurun_out/ktrim/b${nb}_no$v.json 2> gpurun_out/ktrim/b${nb}_no$v.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/ktrim/b${nb}_no$v.json'));print('nb $nb no_ktrim=$v', round(d['kernel_ms'],3),'ms', round(d['value']),'GF/s residual', d.get('residual'))"
done; done
python tools/parity_sweep.py > gpurun_out/ktrim/parity_sweep.log 2>&1; echo sweep_rc=$?; tail -3 gpurun_out/ktrim/parity_sweep.log
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ktrim/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/ktrim/pytest.log
