# smoke() plainly, then under the driver-style ncu launch list (serialised launches)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/smoke_ncu.log
grep -o '"[a-zA-Z_:]*\(exec_kernel\|k_put\|k_get\|k_bsmall\)[^"]*"' gpurun_out/smoke_launches.csv | sort | uniq -c
python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?
tail -c 2500 gpurun_out/bench_c4.json
