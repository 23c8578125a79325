export TINV_PRIO_NORM=0 TINV_CRIT_SLACK=-1
for tb in 0 20 40 80 160; do
export TINV_TAIL_BL=$tb
for w in c2 c1; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
python -c "import json;d=json.load(open('gpurun_out/b_$w.json'));print('tail $tb $w', round(d['kernel_ms'],3))"
done
done
export TINV_TAIL_BL=40
timeout 500 python tools/critpath.py 8192 256 out 2>&1 | grep -E "exec|gaps \(|SYRK_ADD_T ->" | head -4
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
python -c "import json;d=json.load(open('gpurun_out/b_c3.json'));print('tail 40 c3', round(d['kernel_ms'],2))"
