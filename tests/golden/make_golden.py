"""Generate golden fixtures from the LIVE reference package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small fixtures under tests/golden/ that pin the oracle (oracle/) and the
host logic of the product package against the reference's own outputs:

  kernels.npz   random tiles through each reference kernel (kernels.py:59-151)
  streams.json  format_stream text / hashes and DAG statistics for small t
  numeric.npz   per-step and full-inversion outputs on seeded SPD inputs
  errors.json   failing-task ids and tile-local indices (scheduler.py:345-347)
  c1.json       fingerprints at BASELINE config 1 (n=1024, nb=128)

`/root/reference` is read-only and absent on the GPU box; nothing at test time
imports it -- tests read only these committed files.
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tileinv as ti  # noqa: E402
from tileinv import kernels as K  # noqa: E402
from tileinv.dag_analysis import critical_path, hazard_census  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def spd(n, seed=0, shift=1.0):
    g = np.random.default_rng(seed).standard_normal((n, n))
    a = g @ g.T / n + shift * np.eye(n)
    return ti.symmetrize_lower(a)


def kernels_fixture():
    rng = np.random.default_rng(1234)
    out = {}
    for b in (1, 3, 8, 17):
        m = rng.standard_normal((b, b))
        spdt = m @ m.T + b * np.eye(b)
        lo = np.tril(rng.standard_normal((b, b))) + 3 * np.eye(b)
        c, a, bb = (rng.standard_normal((b, b)) for _ in range(3))
        # garbage in the strict upper part must be ignored by triangular kernels
        lo_dirty = lo + np.triu(rng.standard_normal((b, b)), 1)
        spd_dirty = np.tril(spdt) + np.triu(rng.standard_normal((b, b)), 1)
        out[f"b{b}_spd"] = spd_dirty
        out[f"b{b}_lo"] = lo_dirty
        out[f"b{b}_c"] = c
        out[f"b{b}_a"] = a
        out[f"b{b}_b"] = bb
        out[f"b{b}_potrf"] = K.potrf(spd_dirty)
        out[f"b{b}_trsm"] = K.trsm_right_lt(a, lo_dirty)
        out[f"b{b}_syrk_sub"] = K.syrk_sub(c, a)
        out[f"b{b}_syrk_add_t"] = K.syrk_add_t(c, a)
        out[f"b{b}_gemm_nt"] = K.gemm(c, a, bb, False, -1)
        out[f"b{b}_gemm_nn"] = K.gemm(c, a, bb, False, 1)
        out[f"b{b}_gemm_tn"] = K.gemm(c, a, bb, True, 1)
        out[f"b{b}_trtri"] = K.trtri(lo_dirty)
        out[f"b{b}_trmm_left"] = K.trmm_left(a, lo_dirty)
        out[f"b{b}_trmm_right_neg"] = K.trmm_right_neg(a, lo_dirty)
        out[f"b{b}_trmm_left_t"] = K.trmm_left_t(a, lo_dirty)
        out[f"b{b}_lauum"] = K.lauum(lo_dirty)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def variants():
    for pl in (ti.Placement.IN_PLACE, ti.Placement.OUT_OF_PLACE):
        for loops in ("UDU", "UUU", "DDD", "DUD"):
            for pipe in (True, False):
                yield pl, loops, pipe


def streams_fixture():
    res = {"full": {}, "step": {}}
    for t in range(1, 9):
        for pl, loops, pipe in variants():
            s = ti.gen_inversion(t, ti.VariantConfig(pl, loops, pipe))
            txt = ti.format_stream(s)
            dag = ti.build_dag(s)
            rep = critical_path(dag)
            cen = hazard_census(dag)
            key = f"t{t}_{pl.value}_{loops}_{int(pipe)}"
            res["full"][key] = {
                "ntasks": len(s.tasks),
                "sha": hashlib.sha256(txt.encode()).hexdigest(),
                "text": txt if t <= 3 else None,
                "nedges": len(dag.edges),
                "cp": rep.critical_path,
                "cp_copies": rep.copy_inclusive_path,
                "census": {k.value: dict(v) for k, v in cen.items()},
            }
        for d in "UD":
            for step, fn in ((1, None), (2, ti.Placement.IN_PLACE), (2, ti.Placement.OUT_OF_PLACE),
                             (3, ti.Placement.IN_PLACE), (3, ti.Placement.OUT_OF_PLACE)):
                if step == 1:
                    s = ti.gen_step1(t, d)
                    key = f"t{t}_s1_{d}"
                elif step == 2:
                    s = ti.gen_step2(t, d, fn)
                    key = f"t{t}_s2_{fn.value}_{d}"
                else:
                    s = ti.gen_step3(t, d, fn)
                    key = f"t{t}_s3_{fn.value}_{d}"
                txt = ti.format_stream(s)
                dag = ti.build_dag(s)
                res["step"][key] = {
                    "ntasks": len(s.tasks),
                    "sha": hashlib.sha256(txt.encode()).hexdigest(),
                    "text": txt if t <= 3 else None,
                    "nedges": len(dag.edges),
                    "cp": critical_path(dag).critical_path,
                    "edges": sorted([e.src, e.dst, e.kind.value if e.kind else "BAR"] for e in dag.edges)
                    if t <= 3 else None,
                }
    with open(os.path.join(HERE, "streams.json"), "w") as fh:
        json.dump(res, fh, indent=0, sort_keys=True)


def numeric_fixture():
    out = {}
    for n, b in ((64, 16), (120, 40)):
        a = spd(n)
        out[f"n{n}_A"] = a
        t = n // b
        # per-step chain, both placements
        for pl in (ti.Placement.IN_PLACE, ti.Placement.OUT_OF_PLACE):
            tm = ti.from_dense(a, b)
            ti.execute(ti.gen_step1(t, "U"), tm, 2)
            out[f"n{n}_{pl.value}_step1"] = np.tril(ti.to_dense(tm))
            ti.execute(ti.gen_step2(t, "D", pl), tm, 2)
            out[f"n{n}_{pl.value}_step2"] = np.tril(ti.to_dense(tm))
            ti.execute(ti.gen_step3(t, "U", pl), tm, 2)
            out[f"n{n}_{pl.value}_step3"] = ti.to_dense(tm)  # upper tiles keep stale A
        for pl, loops, pipe in variants():
            if loops not in ("UDU", "UUU"):
                continue
            tm = ti.from_dense(a, b)
            ti.execute(ti.gen_inversion(t, ti.VariantConfig(pl, loops, pipe)), tm, 3)
            out[f"n{n}_full_{pl.value}_{loops}_{int(pipe)}"] = ti.symmetrize_lower(ti.to_dense(tm))
    np.savez_compressed(os.path.join(HERE, "numeric.npz"), **out)


def errors_fixture():
    res = {}
    # NPD: make the Schur complement of tile row 2 negative at local index 3
    n, b = 64, 16
    a = spd(n)
    a[2 * b + 3, 2 * b + 3] = -5.0
    for pl in (ti.Placement.IN_PLACE, ti.Placement.OUT_OF_PLACE):
        tm = ti.from_dense(a, b)
        before = ti.to_dense(tm).copy()
        try:
            ti.execute(ti.gen_inversion(4, ti.VariantConfig(pl)), tm, 2)
            res[f"npd_{pl.value}"] = None
        except ti.ExecutionError as e:
            res[f"npd_{pl.value}"] = {"task": e.task.id, "kind": e.task.kind_name,
                                      "indices": list(e.task.indices), "cause": type(e.cause).__name__,
                                      "index": e.cause.index,
                                      "unchanged": bool(np.array_equal(before, ti.to_dense(tm)))}
    np.save(os.path.join(HERE, "npd_A.npy"), a)
    # singular TRTRI: step 2 on a lower factor with an exact zero on the diagonal
    l = np.tril(spd(n))
    l[3 * b + 7, 3 * b + 7] = 0.0
    l[1 * b + 2, 1 * b + 2] = 0.0
    tm = ti.from_dense(l, b)
    try:
        ti.execute(ti.gen_step2(4, "D"), tm, 2)
        res["singular_step2"] = None
    except ti.ExecutionError as e:
        res["singular_step2"] = {"task": e.task.id, "kind": e.task.kind_name,
                                 "indices": list(e.task.indices), "cause": type(e.cause).__name__,
                                 "index": e.cause.index}
    np.save(os.path.join(HERE, "singular_L.npy"), l)
    # singular TRSM: step 1 where POTRF is bypassed -- stream of one TRSM
    with open(os.path.join(HERE, "errors.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)


def c1_fixture():
    n, b = 1024, 128
    a = spd(n)
    tm = ti.from_dense(a, b)
    ti.execute(ti.gen_inversion(n // b, ti.VariantConfig()), tm, 4)
    x = ti.symmetrize_lower(ti.to_dense(tm))
    ref = np.linalg.inv(a)
    res = {
        "A_sha16": hashlib.sha256(a.tobytes()).hexdigest()[:16],
        "X_tril_sha16": hashlib.sha256(np.tril(ti.to_dense(tm)).tobytes()).hexdigest()[:16],
        "X_sum": float(x.sum()), "X_absmax": float(np.abs(x).max()),
        "X_vs_numpy_inv_normwise": float(np.abs(x - ref).max() / np.abs(ref).max()),
        "cond": float(np.linalg.cond(a)),
        "residual": float(np.linalg.norm(np.eye(n) - a @ x, 1)
                          / (n * np.linalg.norm(a, 1) * np.linalg.norm(x, 1) * np.finfo(float).eps)),
    }
    with open(os.path.join(HERE, "c1.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    kernels_fixture()
    streams_fixture()
    numeric_fixture()
    errors_fixture()
    c1_fixture()
    print("golden fixtures written to", HERE)
