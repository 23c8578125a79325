mkdir -p gpurun_out
for lo in UDU UDD; do
python bench.py --workload c2 --loops $lo --steps 10 --warmup 3 --no-cpu --no-load > gpurun_out/c2_$lo.json 2> gpurun_out/c2_$lo.err; echo $lo rc=$?
python -c "import json;d=json.load(open('gpurun_out/c2_$lo.json'));print('$lo', round(d['value']), round(d['kernel_ms'],2), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), d['steps_breakdown']['pipelined_ms'], d['steps_breakdown']['barriered_ms'])"
done
TINV_DEPART_PROFILE=1 python - > gpurun_out/c2_depart.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
from oracle import tileinv_oracle as O
n, b = 8192, 256
a = O.spd_matrix(n, 0, 1.0)
ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy(); ha[...] = a
hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
for lo in ("UDU", "UDD"):
    cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE, lo, True)
    t = n // b
    s = P.gen_inversion(t, cfg)
    ctx = _native.Context(n, b)
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO | _native.TRACE)
    for _ in range(2):
        rc, err, ms = plan.run_host(ha.ctypes.data, n, hx.ctypes.data, n)
    print(lo, rc, ms, file=sys.stderr)
    plan.close(); ctx.close()
PY
cat gpurun_out/c2_depart.log | tail -8
