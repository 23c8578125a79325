# ncu full set with source counters on one k_bpipe launch (2048 x n=256), then the raw/source pages
mkdir -p gpurun_out
timeout 120 python tools/bsmall_probe.py 2048 256 > gpurun_out/probe.log 2>&1; echo probe_rc=$?; tail -2 gpurun_out/probe.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bpipe -s 3 -c 1 -o gpurun_out/bpipe_full2 -f python tools/bsmall_probe.py 2048 256 > gpurun_out/ncu_bpipe.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_bpipe.log
