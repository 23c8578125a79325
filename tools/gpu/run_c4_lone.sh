# C4: uncontended phase spans (1, 2, 3 CTAs per SM) and the inner loop's DMMA rate
mkdir -p gpurun_out/c4lone
./tools/micro/quad_rate > gpurun_out/c4lone/quad_rate.log 2>&1; cat gpurun_out/c4lone/quad_rate.log
for pad in 64 32 0; do
  echo "== pad $pad KB"
  TINV_BSMALL_PAD_KB=$pad TINV_BSMALL_PROF=1 python tools/bsmall_probe.py 8192 256 2>&1 | grep -E "cycles per matrix|median" | tail -3
done | tee gpurun_out/c4lone/phases.log
