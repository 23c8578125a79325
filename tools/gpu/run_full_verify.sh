# round-end style verification: GPU tests, smoke, bench lines for every config, reference arm
mkdir -p gpurun_out/verify
python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=10 > gpurun_out/verify/pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/verify/pytest.log | grep -E "passed|failed|error" 
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/verify/smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/verify/bench_c3.json 2> gpurun_out/verify/bench_c3.err; echo c3_rc=$?
for w in c1 c2 c4; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/verify/bench_$w.json 2> gpurun_out/verify/bench_$w.err; echo ${w}_rc=$?; done
python bench.py --workload c5 --steps 3 --warmup 3 --share-slots > gpurun_out/verify/bench_c5.json 2> gpurun_out/verify/bench_c5.err; echo c5_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/verify/ref.json 2> gpurun_out/verify/ref.err; echo ref_rc=$?
for f in c1 c2 c3 c4 c5; do python -c "
import json;d=json.load(open('gpurun_out/verify/bench_$f.json'));e=d.get('e2e') or {}
print('$f', round(d['value']), 'GF/s', round(d['kernel_ms'],3), 'ms', 'frac', round(d['roofline']['frac'],3), 'e2e', round(e.get('value',0)))"; done
