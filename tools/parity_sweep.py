"""Randomized parity sweep (GPU box): the fused batched engine over many n,
the DAG executor over random (n, nb, placement, loops, pipelining), each
against numpy's inverse (normwise <= 1e-10 cond, residual < 10)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from oracle import tileinv_oracle as O  # noqa: E402

rng = np.random.default_rng(2026)
fails = 0
ns = list(range(1, 17)) + [31, 32, 33, 63, 64, 65, 96, 127, 128, 129, 150, 191, 192, 193, 224, 254, 255, 256]
for n in ns:
    B = int(rng.integers(1, 9))
    shift = float(rng.choice([1.0, 0.1, 1e-3]))
    a = np.stack([O.spd_matrix(n, int(rng.integers(1 << 30)), shift) for _ in range(B)])
    x = P.invert_batched(a, n, engine="fused")
    for k in range(B):
        ref = np.linalg.inv(a[k])
        cond = np.linalg.cond(a[k])
        rel = np.max(np.abs(x[k] - ref)) / np.max(np.abs(ref))
        res = O.residual(a[k], x[k])
        if not (rel <= 1e-10 * cond and res < 10 and np.array_equal(x[k], x[k].T)):
            fails += 1
            print(f"FUSED FAIL n={n} k={k} rel={rel:.2e} cond={cond:.1e} res={res:.2f}")
print(f"fused: {len(ns)} sizes checked", flush=True)
cases = 0
for _ in range(40):
    nb = int(rng.choice([1, 2, 3, 7, 16, 50, 64, 100, 128, 130, 200, 256]))
    t = int(rng.integers(1, 7))
    n = nb * t
    if n > 1200:
        continue
    cfg = P.VariantConfig(P.Placement(rng.choice(["in", "out"])), "".join(rng.choice(list("UD"), 3)),
                          bool(rng.integers(2)))
    a = O.spd_matrix(n, int(rng.integers(1 << 30)), float(rng.choice([1.0, 0.05])))
    x = P.invert(a, nb, cfg)
    ref = np.linalg.inv(a)
    cond = np.linalg.cond(a)
    rel = np.max(np.abs(x - ref)) / np.max(np.abs(ref))
    res = O.residual(a, x)
    cases += 1
    if not (rel <= 1e-10 * cond and res < 10):
        fails += 1
        print(f"DAG FAIL n={n} nb={nb} {cfg} rel={rel:.2e} cond={cond:.1e} res={res:.2f}")
print(f"dag: {cases} random configurations checked; failures total {fails}", flush=True)
sys.exit(1 if fails else 0)
