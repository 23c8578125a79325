mkdir -p gpurun_out
export TINV_PRIO_NORM=0 TINV_CRIT_SLACK=-1 TINV_DUMP_LEVELS=gpurun_out/levels_c2.txt
timeout 500 python tools/critpath.py 8192 256 out gpurun_out/critpath_c2.json 2>&1 | grep -E "exec|gaps \(" | head -3
