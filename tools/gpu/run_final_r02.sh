# final round-2 evidence: full verification, then (each after its plain command exited 0)
# the ncu launch list of the default bench and one full-set capture of exec_kernel at C3
bash tools/gpu/run_full_verify.sh
mkdir -p gpurun_out/ncu_final
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ncu_final/plain_c3.json 2> gpurun_out/ncu_final/plain_c3.err; echo plain_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_final/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-steps --no-load > gpurun_out/ncu_final/launches_c3.log 2>&1; echo ncu_list_rc=$?
python tools/ncu_target.py 32768 512 > gpurun_out/ncu_final/target_plain.log 2>&1; echo target_rc=$?
timeout 2400 ncu --set full --import-source on --clock-control none -k regex:exec_kernel -s 1 -c 1 -o gpurun_out/ncu_final/exec_c3_full -f python tools/ncu_target.py 32768 512 > gpurun_out/ncu_final/exec_c3_full.log 2>&1; echo ncu_full_rc=$?
ls -la gpurun_out/ncu_final
