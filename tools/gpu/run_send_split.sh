mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "separate_stores or distributed or loopback or multi" -p no:cacheprovider > gpurun_out/ranks_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/ranks_tests.log
timeout 1200 python tools/ranks_local.py 32768 512 1,2,4,8 > gpurun_out/ranks_local_c3.log 2> gpurun_out/ranks_local_c3.err; echo rc=$?
cut -c1-260 gpurun_out/ranks_local_c3.log
timeout 900 python tools/emulate_scaling.py > gpurun_out/emulate.log 2>&1; echo emu_rc=$?; tail -5 gpurun_out/emulate.log | cut -c1-300
