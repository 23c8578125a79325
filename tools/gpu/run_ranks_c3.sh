mkdir -p gpurun_out
timeout 1200 python tools/ranks_local.py ${N:-4096} ${NB:-512} ${W:-1,2} > gpurun_out/ranks_local_c3.log 2> gpurun_out/ranks_local_c3.err; echo rc=$?
cat gpurun_out/ranks_local_c3.log; tail -3 gpurun_out/ranks_local_c3.err
