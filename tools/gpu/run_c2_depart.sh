# C2 streamed plan: when do the result tiles become final (TINV_DEPART_PROFILE), per loop order / departure weight
mkdir -p gpurun_out
for w in default 2 8; do
if [ "$w" != default ]; then export TINV_DEPART_WEIGHT=$w; fi
TINV_DEPART_PROFILE=1 timeout 300 python - 2>&1 <<'PY' | grep -E "depart\]|arrive\]|UDU|UDD"
import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
from oracle import tileinv_oracle as O
n, b = 8192, 256
a = O.spd_matrix(n, 0, 1.0)
ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy(); ha[...] = a
hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
for lo in ("UDU",):
    cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE, lo, True)
    t = n // b
    s = P.gen_inversion(t, cfg)
    ctx = _native.Context(n, b)
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO | _native.TRACE)
    for _ in range(3):
        rc, err, ms = plan.run_host(ha.ctypes.data, n, hx.ctypes.data, n)
    print(lo, os.environ.get("TINV_DEPART_WEIGHT", "default"), rc, ms, file=sys.stderr)
    plan.close(); ctx.close()
PY
done
