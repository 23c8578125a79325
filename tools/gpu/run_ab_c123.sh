mkdir -p gpurun_out/ab
for w in c1 c2 c3; do
python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ab/bench_$w.json 2> gpurun_out/ab/bench_$w.err; echo ${w}_rc=$?
python -c "import json;d=json.load(open('gpurun_out/ab/bench_$w.json'));print('$w', round(d['kernel_ms'],3),'ms', round(d['value']),'GF/s frac', round(d['roofline']['frac'],4), 'residual', d.get('residual'))"
done
