"""Randomized soak of the DAG executor on the GPU box: for `minutes` minutes,
random (n, nb, placement, loop orders, pipelining, slot sharing) through three
entry paths -- `invert` (staged), `invert_host` (streamed host I/O) and
`run_in_order` -- each checked against numpy's inverse (normwise <= 1e-10 cond,
residual < 10) and against each other BITWISE (the executor is deterministic
across schedules and paths). Also random failing inputs: the reported task and
tile-local index must equal the oracle's.

  python tools/parity_soak.py [minutes] [seed]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1002_4057_b200 as P  # noqa: E402
from oracle import tileinv_oracle as O  # noqa: E402

minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
deadline = time.time() + 60.0 * minutes
cases = fails = neg = 0
while time.time() < deadline:
    nb = int(rng.choice([1, 2, 5, 8, 16, 33, 64, 72, 100, 128, 130, 136, 200, 256, 384]))
    t = int(rng.integers(1, 13))
    n = nb * t
    if n > 3072 or (nb < 8 and t > 8):
        continue
    cfg = P.VariantConfig(P.Placement(rng.choice(["in", "out"])), "".join(rng.choice(list("UD"), 3)),
                          bool(rng.integers(2)))
    share = bool(rng.integers(2))
    a = O.spd_matrix(n, int(rng.integers(1 << 30)), float(rng.choice([1.0, 0.05, 1e-3])))
    tag = f"n={n} nb={nb} {cfg.placement.value} {cfg.loops} pipelined={cfg.pipelined} share={share}"
    try:
        x = P.invert(a, nb, cfg, share_slots=share)
        xh = np.empty_like(a)
        P.invert_host(a, nb, cfg, out=xh)
        tm = P.from_dense(a, nb)
        P.run_in_order(P.gen_inversion(t, cfg), tm)
        xs = P.to_dense_symmetric(tm)
    except Exception as exc:  # noqa: BLE001
        fails += 1
        print(f"FAIL (exception) {tag}: {exc!r}", flush=True)
        continue
    ref = np.linalg.inv(a)
    cond = np.linalg.cond(a)
    rel = np.max(np.abs(x - ref)) / np.max(np.abs(ref))
    res = O.residual(a, x)
    cases += 1
    ok = rel <= 1e-10 * cond and res < 10 and np.array_equal(x, xh) and np.array_equal(x, xs)
    if not ok:
        fails += 1
        print(f"FAIL {tag}: rel={rel:.2e} cond={cond:.1e} res={res:.2f} host_equal={np.array_equal(x, xh)} "
              f"in_order_equal={np.array_equal(x, xs)}", flush=True)
    if cases % 4 == 0 and t >= 2:  # a failing input: the same task and index as the oracle's POTRF chain
        j = int(rng.integers(n))
        bad = a.copy()
        bad[j, j] = -abs(bad[j, j])
        exp = None
        try:
            O.invert(bad, nb, cfg.loops, cfg.placement == P.Placement.OUT_OF_PLACE, cfg.pipelined)
        except Exception as exc:  # noqa: BLE001
            exp = exc
        got = None
        try:
            P.invert(bad, nb, cfg)
        except P.ExecutionError as exc:
            got = exc
        neg += 1
        same = (exp is not None and got is not None and getattr(exp, "task_id", -1) == got.task.id
                and getattr(getattr(exp, "cause", None), "index", -1) == getattr(got.cause, "index", -2))
        if not same:
            fails += 1
            print(f"FAIL (negative) {tag} j={j}: oracle {exp!r} / device {got!r}", flush=True)
    P.clear_plan_cache()
print(f"soak seed {seed}: {cases} configurations x 3 paths, {neg} failing inputs; failures {fails}", flush=True)
sys.exit(1 if fails else 0)
