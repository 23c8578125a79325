"""Quick GPU sanity: per-tile kernels and one small inversion, verbose."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import kernels as K
from oracle import tileinv_oracle as O

def rel(x, r): return float(np.max(np.abs(x - r)) / max(np.max(np.abs(r)), 1e-300))
print("devices", P._native.device_count() if hasattr(P, "_native") else None, flush=True)
for b in (128, 256):
    rng = np.random.default_rng(b)
    c, a, bb = (rng.standard_normal((b, b)) for _ in range(3))
    m = rng.standard_normal((b, b)); spd = m @ m.T / b + np.eye(b)
    lo = np.tril(rng.standard_normal((b, b))) / np.sqrt(b) + 2 * np.eye(b)
    for name, f, g in [
        ("gemm_nt", lambda: K.gemm(c, a, bb, False, -1), lambda: O.gemm(c, a, bb, False, -1)),
        ("gemm_nn", lambda: K.gemm(c, a, bb, False, 1), lambda: O.gemm(c, a, bb, False, 1)),
        ("gemm_tn", lambda: K.gemm(c, a, bb, True, 1), lambda: O.gemm(c, a, bb, True, 1)),
        ("syrk_sub", lambda: K.syrk_sub(c, a), lambda: O.syrk_sub(c, a)),
        ("syrk_add_t", lambda: K.syrk_add_t(c, a), lambda: O.syrk_add_t(c, a)),
        ("trmm_left", lambda: K.trmm_left(a, lo), lambda: O.trmm_left(a, lo)),
        ("trmm_right_neg", lambda: K.trmm_right_neg(a, lo), lambda: O.trmm_right_neg(a, lo)),
        ("trmm_left_t", lambda: K.trmm_left_t(a, lo), lambda: O.trmm_left_t(a, lo)),
        ("lauum", lambda: K.lauum(lo), lambda: O.lauum(lo)),
        ("potrf", lambda: K.potrf(spd), lambda: O.potrf(spd)),
        ("trtri", lambda: K.trtri(lo), lambda: O.trtri(lo)),
        ("trsm", lambda: K.trsm_right_lt(a, lo), lambda: O.trsm_right_lt(a, lo)),
    ]:
        t0 = time.time()
        try:
            x = f()
            print(f"b={b} {name:15s} rel={rel(x, g()):.3e}  {time.time()-t0:.2f}s", flush=True)
        except Exception as e:
            print(f"b={b} {name:15s} FAILED {type(e).__name__}: {e}", flush=True)
for n, b in ((512, 128), (1024, 256)):
    a = O.spd_matrix(n)
    t0 = time.time()
    x = P.invert(a, b)
    print(f"invert n={n} b={b}: rel={rel(x, np.linalg.inv(a)):.3e} res={O.residual(a, x):.3e} {time.time()-t0:.2f}s", flush=True)
