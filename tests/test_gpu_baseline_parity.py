"""Parity against the reference path at BASELINE.json's large configs.

The reference algorithm is `tileinv.scheduler.execute` over
`tileinv.taskgen.gen_inversion` / `gen_step1/2/3` with the numpy tile kernels
of `tileinv.kernels` (/root/reference/pkg/src/tileinv/scheduler.py:261-351,
taskgen.py:178-269, kernels.py:59-151). Its restatement
`oracle/tileinv_oracle.py` is pinned bitwise to the live reference
(tests/test_oracle.py, tests/golden/); here it runs on the GPU box's host
cores (threaded executor, one worker per core, BLAS 1 thread -- the
reference's fastest mode) on the SAME input bytes the B200 path gets.

* C2 (n=8192, nb=256): A from numpy PCG64 seed 0; the full
  inversion and each step (step k on the oracle's output of step k-1) vs the
  oracle.
* C5 (n=65536, nb=1024, A = G G^T/n + 1e-3 I, cond ~4e3) on one B200: the
  conditioning under which TRSM as a multiply by the explicit L_jj^-1 must
  hold up against the reference's substitution (kernels.py:79-88): normwise
  vs cuSOLVER potrf + potri on the same device, residual on 2048 columns.
* C3 (n=32768, nb=512), once: the bench variant (out-of-place, DDU,
  pipelined) vs the oracle (~150 s on 16 cores; needs ~50 GB of host RAM).

Tolerance (north_star): normwise max|X - R| / max|R| <= 1e-10 * cond(A);
residual ||I - A X||_1 / (n ||A||_1 ||X||_1 eps) = O(1) (< 10).
"""

import os
import time

import numpy as np
import pytest

import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
from oracle import tileinv_oracle as O

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16
CORES = len(os.sched_getaffinity(0))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if _native.device_count() < 1:
        pytest.fail("no B200 visible: the GPU tests must run on the GPU box")


def _avail_ram():
    with open("/proc/meminfo") as fh:
        return next(int(l.split()[1]) * 1024 for l in fh if l.startswith("MemAvailable"))


def _oracle(stream, store):
    """oracle execute (scheduler.py:261-351 restated), every host core, BLAS 1 thread."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1, "blas"):
        return O.execute(stream, store, workers=CORES)


def _tiles_normwise(x_dense, store, n, b, label="A", full_diag=True):
    """max |X - R| / max |R| over the authoritative lower tiles (tile by tile,
    no n x n temporaries); strictly-upper parts of diagonal tiles included only
    when the step leaves them defined (steps 1-2: zero; step 3: symmetric)."""
    t = n // b
    num = den = 0.0
    for i in range(t):
        for j in range(i + 1):
            r = store[(label, i, j)]
            x = x_dense[i * b:(i + 1) * b, j * b:(j + 1) * b]
            if i == j and not full_diag:
                r, x = np.tril(r), np.tril(x)
            num = max(num, float(np.max(np.abs(x - r))))
            den = max(den, float(np.max(np.abs(r))))
    return num / den


def _cond1(a, x):
    """1-norm condition estimate ||A||_1 ||A^-1||_1 from the computed inverse."""
    return float(np.abs(a).sum(0).max() * np.abs(x).sum(0).max())


def _residual_cols(a, x, cols):
    n = a.shape[0]
    r = a @ x[:, cols]
    r[cols, np.arange(len(cols))] -= 1.0
    return float(np.abs(r).sum(0).max() / (n * np.abs(a).sum(0).max() * np.abs(x).sum(0).max() * EPS))


@pytest.fixture(scope="module")
def c2_input():
    return O.spd_matrix(8192, 0, 1.0)  # numpy PCG64 seed 0, SURVEY.md §8(d) recipe


def test_c2_full_inversion_vs_oracle(c2_input):
    """BASELINE config 2, reference default VariantConfig() (in-place, UDU,
    pipelined): P.invert vs oracle execute(gen_inversion) (scheduler.py:261)."""
    a, n, b = c2_input, 8192, 256
    x = P.invert(a, b)
    st = _oracle(O.gen_stream(n // b, (1, 2, 3), "UDU", False, True), O.lower_tiles(a, b))
    cond = _cond1(a, x)
    err = _tiles_normwise(x, st, n, b)
    print(f"C2 full: normwise vs oracle {err:.3e} (tol {1e-10 * cond:.2e})")
    assert err <= 1e-10 * cond, (err, cond)
    cols = np.random.default_rng(1).choice(n, 256, replace=False)
    assert _residual_cols(a, x, cols) < 10


def test_c2_each_step_vs_oracle(c2_input):
    """BASELINE config 2's per-step entry points, each on the oracle's output of
    the previous step: gen_step1 "U" (taskgen.py:230), gen_step2 "D"
    (taskgen.py:236), gen_step3 "U" (taskgen.py:245), in place."""
    a, n, b = c2_input, 8192, 256
    t = n // b
    x_inv = P.invert(a, b)
    cond = _cond1(a, x_inv)
    del x_inv
    src = a
    st = O.lower_tiles(a, b)
    for step, d in ((1, "U"), (2, "D"), (3, "U")):
        gen = {1: lambda: P.gen_step1(t, d), 2: lambda: P.gen_step2(t, d), 3: lambda: P.gen_step3(t, d)}[step]
        tm = P.from_dense(src, b)
        P.execute(gen(), tm)
        x = P.to_dense(tm)
        st = _oracle(O.gen_stream(t, (step,), d, False, True), st)
        err = _tiles_normwise(x, st, n, b, full_diag=(step == 3))
        print(f"C2 step {step} ({d}): normwise vs oracle {err:.3e} (tol {1e-10 * cond:.2e})")
        assert err <= 1e-10 * cond, (step, err, cond)
        # next step's input: the oracle's output (lower tiles), same bytes for both paths
        src = O.assemble_lower(st, n, b)
        if step == 2:
            src = np.tril(src)


def test_c5_conditioning_vs_cusolver_one_gpu():
    """BASELINE config 5 on one B200 (the config names 8; the arithmetic is the
    same per tile): A = G G^T/n + 1e-3 I, n=65536, nb=1024, cond ~4e3."""
    import torch

    n, b = 65536, 1024
    free, _ = torch.cuda.mem_get_info()
    if free < 140e9:
        pytest.skip(f"C5 needs ~140 GB of free HBM, {free / 1e9:.0f} GB free")
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = torch.empty(n, n, dtype=torch.float64, device="cuda")
    blk = 8192  # A = G G^T / n in row blocks of G (G itself: 34 GB)
    g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
    for r in range(0, n, blk):
        torch.matmul(g[r:r + blk], g.T, out=a[r:r + blk])
    del g
    a.div_(n)
    a.diagonal().add_(1e-3)
    for r in range(0, n, blk):  # mirror the lower triangle (bitwise symmetric A), block by block
        d = a[r:r + blk, r:r + blk]
        d.copy_(torch.tril(d) + torch.tril(d, -1).T)
        a[:r, r:r + blk] = a[r:r + blk, :r].T
    torch.cuda.empty_cache()
    t = n // b
    cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True)
    ctx = _native.Context(n, b)
    s = P.gen_inversion(t, cfg)
    # memory-constrained renaming: C reuses B's slots (store 4T -> 3T tiles, 71.6 -> 53.6 GB at C5)
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.SHARE_SLOTS)
    assert plan.rc == 0, plan.msg
    ctx.put_dense_device(a.data_ptr(), n)
    rc, err, ms = plan.run()
    assert rc == 0, plan.msg
    plan.close()
    store = ctx.store_bytes()
    assert store < 60e9
    x = torch.empty_like(a)
    ctx.get_dense_device(x.data_ptr(), n, _native.DENSE_SYMMETRIZE)
    ctx.close()
    torch.cuda.empty_cache()
    cols = torch.randperm(n, device="cuda", generator=torch.Generator("cuda").manual_seed(1))[:2048]
    r = a @ x[:, cols]
    r[cols, torch.arange(len(cols), device="cuda")] -= 1.0
    res = float(r.abs().sum(0).max() / (n * a.abs().sum(0).max() * x.abs().sum(0).max() * EPS))
    del r
    assert res < 10, res
    # Independent FP64 reference: blocked Cholesky / inverse with cuSOLVER
    # potrf on 8192 diagonal blocks and cuBLAS trsm (SUBSTITUTION, as the
    # reference's trsm_right_lt, kernels.py:79-88) + gemm for the rest.
    # torch.linalg.cholesky on the whole n=65536 matrix faults in cuSOLVER
    # (illegal address: > 2^31 elements), hence the blocking.
    ref = _blocked_spd_inverse(a, 8192)
    cond = float(a.abs().sum(0).max() * ref.abs().sum(0).max())
    assert cond > 1e3  # the config's hard conditioning (~4e3 in the 2-norm; the 1-norm estimate is larger)
    rel = float((x - ref).abs().max() / ref.abs().max())
    print(f"C5 1-GPU: exec {ms:.0f} ms (store {store / 1e9:.1f} GB), normwise vs blocked cuSOLVER/cuBLAS {rel:.3e} (tol {1e-10 * cond:.2e}), "
          f"residual(2048 cols) {res:.3e}, cond1 {cond:.3e}")
    assert rel <= 1e-10 * cond


def _blocked_spd_inverse(a, B):
    """A^-1 = L^-T L^-1 by B x B blocks: L (right-looking, potrf + trsm by
    substitution + gemm), L^-1 (block forward substitution), the lower part of
    L^-T L^-1 mirrored. Returns a new n x n tensor; `a` is not modified."""
    import torch

    n = a.shape[0]
    T = n // B
    blk = lambda m, i, j: m[i * B:(i + 1) * B, j * B:(j + 1) * B]  # noqa: E731
    w = torch.tril(a)  # working store: L
    for k in range(T):
        blk(w, k, k).copy_(torch.linalg.cholesky(blk(w, k, k)))
        lkk = blk(w, k, k)
        for i in range(k + 1, T):  # X L_kk^T = A_ik  (triangular solve, not a multiply by an inverse)
            blk(w, i, k).copy_(torch.linalg.solve_triangular(lkk.T, blk(w, i, k), upper=True, left=False))
        for i in range(k + 1, T):
            for j in range(k + 1, i + 1):
                blk(w, i, j).sub_(blk(w, i, k) @ blk(w, j, k).T)
        if a.is_cuda:
            torch.cuda.synchronize()
    v = torch.zeros_like(a)  # L^-1, block column by block column
    eye = torch.eye(B, dtype=a.dtype, device=a.device)
    for j in range(T):
        blk(v, j, j).copy_(torch.linalg.solve_triangular(blk(w, j, j), eye, upper=False))
        for i in range(j + 1, T):
            acc = sum(blk(w, i, k) @ blk(v, k, j) for k in range(j, i))
            blk(v, i, j).copy_(-torch.linalg.solve_triangular(blk(w, i, i), acc, upper=False))
        if a.is_cuda:
            torch.cuda.synchronize()
    del w
    torch.cuda.empty_cache()
    x = torch.empty_like(a)
    for i in range(T):  # X_ij = sum_{k >= i} V_ki^T V_kj, j <= i
        for j in range(i + 1):
            blk(x, i, j).copy_(sum(blk(v, k, i).T @ blk(v, k, j) for k in range(i, T)))
            if j < i:
                blk(x, j, i).copy_(blk(x, i, j).T)
        if a.is_cuda:
            torch.cuda.synchronize()
    for i in range(T):  # diagonal blocks: mirror their lower triangles
        db = blk(x, i, i)
        db.copy_(torch.tril(db) + torch.tril(db, -1).T)
    return x


@pytest.mark.skipif(os.environ.get("TINV_SKIP_C3_ORACLE") == "1", reason="TINV_SKIP_C3_ORACLE=1")
def test_c3_vs_oracle_once():
    """BASELINE config 3 (the bench workload) against the oracle port of the
    reference, same input bytes: ~150 s of host compute on 16 cores."""
    import torch

    n, b = 32768, 512
    if _avail_ram() < 60e9:
        pytest.skip(f"C3 oracle needs ~60 GB of host RAM, {_avail_ram() / 1e9:.0f} GB available")
    gen = torch.Generator(device="cuda").manual_seed(0)
    g = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=gen)
    ad = torch.matmul(g, g.T)
    del g
    ad.div_(n)
    ad.diagonal().add_(1.0)
    ad = torch.tril(ad) + torch.tril(ad, -1).T
    a = ad.cpu().numpy()
    del ad
    torch.cuda.empty_cache()
    cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE, "DDU", True)
    t0 = time.perf_counter()
    x = P.invert(a, b, cfg)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    st = _oracle(O.gen_stream(n // b, (1, 2, 3), "DDU", True, True), O.lower_tiles(a, b))
    t_cpu = time.perf_counter() - t0
    cond = _cond1(a, x)
    err = _tiles_normwise(x, st, n, b)
    print(f"C3 vs oracle: normwise {err:.3e} (tol {1e-10 * cond:.2e}, cond1 {cond:.3e}); "
          f"B200 invert() {t_gpu:.1f} s incl. host copies, oracle {t_cpu:.1f} s on {CORES} cores")
    assert err <= 1e-10 * cond
