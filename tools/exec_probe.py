"""Executor probes: raw GEMM-item throughput on independent-task streams and
per-kind task durations of the full inversion (device trace)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native

n, b = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, int(sys.argv[2]) if len(sys.argv) > 2 else 512
t = n // b
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.T / n
a.diagonal().add_(1.0)
del g
ctx = _native.Context(n, b)

def row(kind, step, out, reads):
    r = [-1] * 16
    r[0], r[1] = kind, step
    r[5:9] = [0, out[0], out[1], 1]
    r[9] = len(reads)
    for x, (i, j) in enumerate(reads):
        r[10 + 3 * x:13 + 3 * x] = [0, i, j]
    return r

def run(table, label, flops):
    table = np.array(table, dtype=np.int32)
    plan = _native.Plan(ctx, table, t, np.zeros(0, np.int64))
    ms = []
    for _ in range(2):
        ctx.put_dense_device(a.data_ptr(), n)
        rc, err, m = plan.run()
        assert rc == 0, plan.msg
        ms.append(m)
    st = plan.stats()
    print(f"{label:40s} {min(ms):9.2f} ms  {flops / min(ms) / 1e9:8.2f} TF/s  ({flops / min(ms) / 1e9 / 37.07 * 100:5.1f}%)  items {st['items']}", flush=True)
    plan.close()

# independent GEMMs: out (i,j) i>j>=1 reading (i,0),(j,0)
pairs = [(i, j) for i in range(2, t) for j in range(1, i)]
for step, name in ((1, "NT"), (2, "NN"), (3, "TN")):
    tab = [row(5, step, (i, j), [(i, 0), (j, 0)]) for i, j in pairs]
    run(tab, f"independent GEMM {name} x{len(pairs)}", 2.0 * b ** 3 * len(pairs))
if len(sys.argv) > 3 and sys.argv[3] == "gemm":
    sys.exit(0)
# chains: 8 GEMMs accumulating into each output (like step-1 updates)
deep = [(i, j) for i, j in pairs if j > 8][:400]
tab = [row(5, 1, (i, j), [(i, k), (j, k)]) for k in range(0, 8) for i, j in deep]
run(tab, "GEMM NT 8-deep chains x400", 2.0 * b ** 3 * len(tab))
# other multi-item kinds, independent
trmm = [row(7, 2, (i, j), [(i, i)]) for i, j in pairs]
run(trmm, "independent TRMM_LEFT", 1.0 * b ** 3 * len(trmm))
syrk = [row(3, 1, (i, i), [(i, j)]) for i in range(1, t) for j in [0]]
run(syrk, "independent SYRK_SUB", 1.0 * b ** 3 * len(syrk))
lau = [row(10, 3, (i, i), []) for i in range(t)]
run(lau, "independent LAUUM", b ** 3 / 3 * len(lau))
pot = [row(1, 1, (i, i), []) for i in range(t)]
run(pot, "independent POTRF (single CTA each)", b ** 3 / 3 * len(pot))
tri = [row(6, 2, (i, i), []) for i in range(t)]
run(tri, "independent TRTRI (single CTA each)", b ** 3 / 3 * len(tri))
# POTRF chain latency: t POTRFs serialized on one tile? use SERIAL on independent tiles
plan = _native.Plan(ctx, np.array(pot[:8], np.int32), t, np.zeros(0, np.int64), _native.SERIAL)
ctx.put_dense_device(a.data_ptr(), n); rc, err, m = plan.run(); plan.close()
print(f"8 POTRF serialized: {m:.2f} ms -> {m/8*1e3:.0f} us per POTRF(b={b})", flush=True)
plan = _native.Plan(ctx, np.array(tri[:8], np.int32), t, np.zeros(0, np.int64), _native.SERIAL)
ctx.put_dense_device(a.data_ptr(), n); rc, err, m = plan.run(); plan.close()
print(f"8 TRTRI serialized: {m:.2f} ms -> {m/8*1e3:.0f} us per TRTRI(b={b})", flush=True)
gem = [row(5, 1, (i, j), [(i, 0), (j, 0)]) for i, j in pairs[:8]]
plan = _native.Plan(ctx, np.array(gem, np.int32), t, np.zeros(0, np.int64), _native.SERIAL)
ctx.put_dense_device(a.data_ptr(), n); rc, err, m = plan.run(); plan.close()
print(f"8 GEMM serialized: {m:.2f} ms -> {m/8*1e3:.0f} us per GEMM task (16 items in parallel)", flush=True)

# full inversion trace
for pl in ("out", "in"):
    s = P.gen_inversion(t, P.VariantConfig(P.Placement(pl)))
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.TRACE)
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, m = plan.run()
    st, en, sm = plan.trace()
    kinds = s.table()[:, 0]
    names = ["COPY", "POTRF", "TRSM", "SYRK_SUB", "SYRK_ADD_T", "GEMM", "TRTRI", "TRMM_LEFT", "TRMM_RIGHT_NEG", "TRMM_LEFT_T", "LAUUM"]
    print(f"full {pl}: {m:.1f} ms", flush=True)
    for k in range(11):
        sel = kinds == k
        if sel.sum() == 0: continue
        d = (en[sel] - st[sel]) / 1e3
        print(f"   {names[k]:15s} n={sel.sum():6d} task span us: mean {d.mean():8.1f} p50 {np.median(d):8.1f} max {d.max():8.1f}", flush=True)
    # busy profile: number of tasks in flight over 20 buckets
    T = en.max()
    edges = np.linspace(0, T, 21)
    prof = []
    for lo, hi in zip(edges[:-1], edges[1:]):
        prof.append(int(((st < hi) & (en > lo)).sum()))
    print("   tasks in flight per 5% bucket:", prof, flush=True)
    plan.close()
