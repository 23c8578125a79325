for pad in 64 0; do
  echo "== pad $pad KB"
  TINV_BSMALL_PAD_KB=$pad TINV_BSMALL_PROF=1 python tools/bsmall_probe.py 8192 256 2>&1 | grep -E "cycles per matrix|median" | tail -3
done
