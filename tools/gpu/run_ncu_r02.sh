# round-2 ncu evidence: launch list of the default bench (C3), C2 exec_kernel full set, C4 k_bsmall key metrics
mkdir -p gpurun_out/ncu
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ncu/plain_c3.json 2>&1; echo plain_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ncu/launches_c3.log 2>&1; echo ncu1_rc=$?
python bench.py --workload c2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ncu/plain_c2.json 2>&1; echo plain2_rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:exec_kernel -s 1 -c 1 -o gpurun_out/ncu/exec_c2_full -f python bench.py --workload c2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ncu/exec_c2_full.log 2>&1; echo ncu2_rc=$?
python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu/plain_c4.json 2>&1; echo plain4_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,smsp__pcsamp_warps_issue_stalled_no_instructions --clock-control none -k regex:k_bsmall -c 3 --csv --log-file gpurun_out/ncu/bsmall_c4.csv python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu/bsmall_c4.log 2>&1; echo ncu4_rc=$?
