# C2 loop orders: kernel time, streamed e2e, steps breakdown
mkdir -p gpurun_out
for lo in UUU UUD; do
timeout 300 python bench.py --workload c2 --loops $lo --steps 10 --warmup 3 --no-cpu --no-load > gpurun_out/c2_$lo.json 2> gpurun_out/c2_$lo.err; echo $lo rc=$?
python -c "import json;d=json.load(open('gpurun_out/c2_$lo.json'));print('$lo', round(d['value']), round(d['kernel_ms'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), d['steps_breakdown']['pipelined_ms'], d['steps_breakdown']['barriered_ms'])"
done
