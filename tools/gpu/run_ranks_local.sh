# every rank in one process: separate (optionally partitioned) stores, concurrent executors, SENDs into peer stores
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "separate_stores or distributed or loopback" -p no:cacheprovider > gpurun_out/ranks_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/ranks_tests.log
