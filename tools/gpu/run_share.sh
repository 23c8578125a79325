mkdir -p gpurun_out
python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "share_slots or c5" > gpurun_out/pytest_share.log 2>&1; echo pytest_rc=$?
grep -E "C5|passed|failed|Error" gpurun_out/pytest_share.log | head
for f in "" "--share-slots"; do
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu --no-steps --no-e2e --no-load $f > gpurun_out/bench_c5$f.json 2> gpurun_out/bench_c5$f.err; echo c5_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c5$f.json'));print(d['value'],d['kernel_ms'],d['store_bytes']/1e9,d['share_slots'],d['residual'])"
done
