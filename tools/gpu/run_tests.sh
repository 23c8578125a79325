set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv; free -g; nproc; lscpu | grep "Model name"
python -m pytest tests -m gpu -q -s -p no:cacheprovider -rs --durations=15 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
tail -60 gpurun_out/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo ncu_rc=$?
tail -5 gpurun_out/ncu_smoke.log
