mkdir -p gpurun_out
timeout 900 python tools/emulate_scaling.py > gpurun_out/emulate_udu.log 2>&1; echo emu_rc=$?
tail -1 gpurun_out/emulate_udu.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(r['ranks'], round(r['kernel_ms'],1), round(r['emulated_efficiency'],3), r['busy_max_over_mean'], r['bitwise_equal_1rank']) for r in d['rows']]"
timeout 900 python tools/emulate_scaling.py --n 8192 --nb 256 --ranks 1,2,4,8 > gpurun_out/emulate_c2.log 2>&1; echo emu2_rc=$?
tail -1 gpurun_out/emulate_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(r['ranks'], round(r['kernel_ms'],2), round(r['emulated_efficiency'],3), r['bitwise_equal_1rank']) for r in d['rows']]"
