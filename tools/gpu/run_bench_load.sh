mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c3.json'));print(d['value'],d['kernel_ms'],json.dumps(d.get('load')))"
tail -3 gpurun_out/bench_c3.err
python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['value'],d['kernel_ms'],d['e2e']['value'],json.dumps(d.get('load')))"
