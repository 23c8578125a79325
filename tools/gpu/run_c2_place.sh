for pl in out in; do for lo in UDU UUD DUU; do
timeout 300 python bench.py --workload c2 --placement $pl --loops $lo --steps 10 --warmup 3 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$pl $lo', round(d['kernel_ms'],3))" 2>/dev/null || tail -2 gpurun_out/b.err
done; done
