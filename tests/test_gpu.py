"""Parity of the B200 path against the oracle and the reference's golden
vectors. Runs on the GPU box (pytest -m gpu); every call goes through the
C-ABI library (libtileinv_b200.so).

Tolerances (BASELINE.json north_star, SURVEY.md §8(d) finding 12):
  * inversion / per-step outputs: normwise max|X-R|/max|R| <= 1e-10 * cond(A)
    and residual ||I - A X||_1 / (n ||A||_1 ||X||_1 eps) = O(1) (< 10);
  * single tile kernels vs the reference kernels: <= 1e-12 relative
    normwise;
  * schedule independence: bitwise.
"""

import json
import os

import numpy as np
import pytest

import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
from paper_1002_4057_b200 import kernels as K
from oracle import tileinv_oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(x, r):
    return float(np.max(np.abs(x - r)) / max(np.max(np.abs(r)), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if _native.device_count() < 1:
        pytest.fail("no B200 visible: the GPU tests must run on the GPU box")


# ---------------------------------------------------------------- tile kernels
@pytest.mark.parametrize("b", [1, 3, 8, 17])
def test_tile_kernels_vs_reference_golden(b):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    f = lambda k: g[f"b{b}_{k}"]  # noqa: E731
    spd, lo, c, a, bb = f("spd"), f("lo"), f("c"), f("a"), f("b")
    tol = 1e-12
    assert rel(K.potrf(spd), f("potrf")) < tol
    assert rel(K.trsm_right_lt(a, lo), f("trsm")) < tol
    assert rel(K.syrk_sub(c, a), f("syrk_sub")) < tol
    assert rel(K.syrk_add_t(c, a), f("syrk_add_t")) < tol
    assert rel(K.gemm(c, a, bb, False, -1), f("gemm_nt")) < tol
    assert rel(K.gemm(c, a, bb, False, 1), f("gemm_nn")) < tol
    assert rel(K.gemm(c, a, bb, True, 1), f("gemm_tn")) < tol
    assert rel(K.trtri(lo), f("trtri")) < tol
    assert rel(K.trmm_left(a, lo), f("trmm_left")) < tol
    assert rel(K.trmm_right_neg(a, lo), f("trmm_right_neg")) < tol
    assert rel(K.trmm_left_t(a, lo), f("trmm_left_t")) < tol
    assert rel(K.lauum(lo), f("lauum")) < tol


@pytest.mark.parametrize("b", [64, 128, 200, 256, 512])
def test_tile_kernels_vs_oracle(b):
    rng = np.random.default_rng(b)
    m = rng.standard_normal((b, b))
    spd = m @ m.T / b + np.eye(b)
    lo = np.tril(rng.standard_normal((b, b))) / np.sqrt(b) + 2 * np.eye(b)
    lo_dirty = lo + np.triu(rng.standard_normal((b, b)), 1)
    c, a, bb = (rng.standard_normal((b, b)) for _ in range(3))
    tol = 1e-12
    assert rel(K.potrf(spd + np.triu(rng.standard_normal((b, b)), 1)), O.potrf(spd)) < tol
    assert rel(K.trsm_right_lt(a, lo_dirty), O.trsm_right_lt(a, lo)) < tol
    assert rel(K.syrk_sub(c, a), O.syrk_sub(c, a)) < tol
    assert rel(K.syrk_add_t(c, a), O.syrk_add_t(c, a)) < tol
    for ta, sg in ((False, -1), (False, 1), (True, 1)):
        assert rel(K.gemm(c, a, bb, ta, sg), O.gemm(c, a, bb, ta, sg)) < tol
    assert rel(K.trtri(lo_dirty), O.trtri(lo)) < tol
    assert rel(K.trmm_left(a, lo_dirty), O.trmm_left(a, lo)) < tol
    assert rel(K.trmm_right_neg(a, lo_dirty), O.trmm_right_neg(a, lo)) < tol
    assert rel(K.trmm_left_t(a, lo_dirty), O.trmm_left_t(a, lo)) < tol
    assert rel(K.lauum(lo_dirty), O.lauum(lo)) < tol
    # output structure: strict upper zero for POTRF / TRTRI, symmetric LAUUM / SYRK
    assert not np.triu(K.potrf(spd), 1).any()
    assert not np.triu(K.trtri(lo_dirty), 1).any()
    s = K.syrk_add_t(c, a)
    assert np.array_equal(s, s.T)


def test_tile_kernel_errors():
    with pytest.raises(K.NotPositiveDefiniteError) as ei:
        K.potrf(np.array([[1.0, 0.0], [2.0, 1.0]]))
    assert ei.value.index == 1
    a = np.eye(300) * 4
    a[257, 257] = -1.0
    with pytest.raises(K.NotPositiveDefiniteError) as ei:
        K.potrf(a)
    assert ei.value.index == 257
    l = np.eye(200)
    l[150, 150] = 0.0
    l[170, 170] = 0.0
    with pytest.raises(K.SingularTileError) as ei:
        K.trtri(l)
    assert ei.value.index == 150
    with pytest.raises(K.SingularTileError) as ei:
        K.trsm_right_lt(np.ones((200, 200)), l)
    assert ei.value.index == 150


# ---------------------------------------------------------------- golden numerics
def _tile_mask(n, b):
    t = n // b
    m = np.zeros((n, n), bool)
    for i in range(t):
        for j in range(i + 1):
            m[i * b:(i + 1) * b, j * b:(j + 1) * b] = True
    return m


@pytest.mark.parametrize("n,b", [(64, 16), (120, 40)])
def test_steps_and_inversions_vs_reference_golden(n, b):
    g = np.load(os.path.join(GOLD, "numeric.npz"))
    a = g[f"n{n}_A"]
    t = n // b
    tol = 1e-10 * np.linalg.cond(a)
    mask = _tile_mask(n, b)
    for pl in P.Placement:
        tm = P.from_dense(a, b)
        P.execute(P.gen_step1(t, "U"), tm)
        x1 = P.to_dense(tm)
        assert rel(np.tril(x1), g[f"n{n}_{pl.value}_step1"]) < tol
        assert np.array_equal(x1[~mask], a[~mask])  # upper tiles stay stale A
        P.execute(P.gen_step2(t, "D", pl), tm)
        assert rel(np.tril(P.to_dense(tm)), g[f"n{n}_{pl.value}_step2"]) < tol
        P.execute(P.gen_step3(t, "U", pl), tm)
        x3 = P.to_dense(tm)
        r3 = g[f"n{n}_{pl.value}_step3"]
        assert rel(x3[mask], r3[mask]) < tol
        assert np.array_equal(x3[~mask], r3[~mask])
    for pl in P.Placement:
        for loops in ("UDU", "UUU"):
            for pipe in (True, False):
                tm = P.from_dense(a, b)
                P.execute(P.gen_inversion(t, P.VariantConfig(pl, loops, pipe)), tm)
                x = P.symmetrize_lower(P.to_dense(tm))
                assert rel(x, g[f"n{n}_full_{pl.value}_{loops}_{int(pipe)}"]) < tol
                assert O.residual(a, x) < 10


def test_errors_vs_reference_golden():
    with open(os.path.join(GOLD, "errors.json")) as fh:
        g = json.load(fh)
    a = np.load(os.path.join(GOLD, "npd_A.npy"))
    for pl in P.Placement:
        tm = P.from_dense(a, 16)
        before = P.to_dense(tm)
        with pytest.raises(P.ExecutionError) as ei:
            P.execute(P.gen_inversion(4, P.VariantConfig(pl)), tm, workers=3)
        exp = g[f"npd_{pl.value}"]
        assert ei.value.task.id == exp["task"]
        assert str(ei.value.task).startswith(exp["kind"])
        assert isinstance(ei.value.cause, P.NotPositiveDefiniteError)
        assert ei.value.cause.index == exp["index"]
        assert np.array_equal(P.to_dense(tm), before)  # a unchanged on failure
    l = np.load(os.path.join(GOLD, "singular_L.npy"))
    tm = P.from_dense(l, 16)
    with pytest.raises(P.ExecutionError) as ei:
        P.execute(P.gen_step2(4, "D"), tm)
    assert ei.value.task.id == g["singular_step2"]["task"]
    assert isinstance(ei.value.cause, P.SingularTileError)
    assert ei.value.cause.index == g["singular_step2"]["index"]


def _stream(t, specs):
    """TaskStream from (kind, step, indices, reads, out) tuples on label A."""
    tasks = []
    for tid, (kind, step, idx, reads, out) in enumerate(specs):
        acc = tuple(P.Access(P.TileId("A", *r), P.Mode.READ) for r in reads)
        acc += (P.Access(P.TileId("A", *out), P.Mode.READWRITE),)
        tasks.append(P.Task(tid, kind, idx, acc, step))
    return P.TaskStream(tasks, set(), t)


def test_failure_after_device_run_restores_device_state():
    # run 1 succeeds and leaves the device copy authoritative (host stale);
    # run 2 fails -> `a` must hold exactly the run-1 result (scheduler.py:345-351)
    n, b = 256, 64
    a = O.spd_matrix(n)
    k = P.KernelKind
    run1 = _stream(4, [(k.SYRK_SUB, P.Step.CHOLESKY, (1, 0), [(1, 0)], (1, 1))] * 50)
    run2 = _stream(4, [(k.POTRF, P.Step.CHOLESKY, (1,), [], (1, 1))])
    twin = P.from_dense(a, b)
    P.execute(run1, twin)
    expect = P.to_dense(twin)
    tm = P.from_dense(a, b)
    P.execute(run1, tm)
    with pytest.raises(P.ExecutionError) as ei:
        P.execute(run2, tm)
    assert isinstance(ei.value.cause, P.NotPositiveDefiniteError)
    assert np.array_equal(P.to_dense(tm), expect)


# ---------------------------------------------------------------- BASELINE config 1 and larger
def test_config1_full_and_steps_vs_oracle():
    n, b = 1024, 128
    a = O.spd_matrix(n, 0, 1.0)
    cond = np.linalg.cond(a)
    ref = O.invert(a, b)
    x = P.invert(a, b)
    assert rel(x, ref) <= 1e-10 * cond
    assert O.residual(a, x) < 10
    st = O.run_in_order(O.gen_stream(8, (1,), "U"), O.lower_tiles(a, b))
    tm = P.from_dense(a, b)
    P.execute(P.gen_step1(8, "U"), tm)
    assert rel(np.tril(P.to_dense(tm)), O.assemble_lower(st, n, b)) <= 1e-10 * cond
    st = O.run_in_order(O.gen_stream(8, (2,), "D"), st)
    P.execute(P.gen_step2(8, "D"), tm)
    assert rel(np.tril(P.to_dense(tm)), O.assemble_lower(st, n, b)) <= 1e-10 * cond
    st = O.run_in_order(O.gen_stream(8, (3,), "U"), st)
    P.execute(P.gen_step3(8, "U"), tm)
    assert rel(P.to_dense(tm)[_tile_mask(n, b)], O.assemble_lower(st, n, b)[_tile_mask(n, b)]) <= 1e-10 * cond


@pytest.mark.parametrize("n,b", [(1024, 256), (2048, 512), (2048, 1024), (1536, 384), (1000, 200)])
def test_larger_tiles_vs_numpy(n, b):
    a = O.spd_matrix(n, 1, 1e-2)
    x = P.invert(a, b, P.VariantConfig(P.Placement.OUT_OF_PLACE))
    ref = np.linalg.inv(a)
    assert rel(x, ref) <= 1e-10 * np.linalg.cond(a)
    assert O.residual(a, x) < 10


def test_variants_and_determinism():
    n, b = 768, 96
    a = O.spd_matrix(n, 3, 0.5)
    ref = O.invert(a, b)
    outs = []
    for pl in P.Placement:
        for loops in ("UDU", "UUU", "DDD"):
            for pipe in (True, False):
                x = P.invert(a, b, P.VariantConfig(pl, loops, pipe))
                assert rel(x, ref) < 1e-12
                outs.append(x)
    # bitwise determinism: repeated runs and sequential replay
    s = P.gen_inversion(8, P.VariantConfig(P.Placement.OUT_OF_PLACE))
    runs = []
    for _ in range(3):
        tm = P.from_dense(a, b)
        P.execute(s, tm)
        runs.append(P.to_dense(tm))
    tm = P.from_dense(a, b)
    P.run_in_order(s, tm)
    runs.append(P.to_dense(tm))
    for r in runs[1:]:
        assert np.array_equal(r, runs[0])


@pytest.mark.parametrize("ticket,prefetch", [("1", "0"), ("3", "0"), ("64", "1"), ("1", "2")])
def test_scheduler_claim_modes_bitwise(monkeypatch, ticket, prefetch):
    # fetch-and-add tickets on every level (overshooting tails, tickets past a
    # level's capacity) and ahead-of-time claims must run every item exactly
    # once: the result is bitwise the default schedule's
    n, b = 1536, 128
    a = O.spd_matrix(n, 6, 0.5)
    cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE)
    base = P.invert(a, b, cfg)
    monkeypatch.setenv("TINV_TICKET_MIN", ticket)
    monkeypatch.setenv("TINV_PREFETCH_MIN", prefetch)
    for _ in range(2):
        assert np.array_equal(P.invert(a, b, cfg), base)
    xb = P.invert_batched(np.stack([a[:256, :256]] * 40), 128)
    monkeypatch.delenv("TINV_TICKET_MIN")
    monkeypatch.delenv("TINV_PREFETCH_MIN")
    assert np.array_equal(xb, P.invert_batched(np.stack([a[:256, :256]] * 40), 128))


def test_layout_roundtrip_and_trace(tmp_path):
    n, b = 640, 160
    a = np.random.default_rng(5).standard_normal((n, n))
    tm = P.from_dense(a, b)
    tm._device()
    tm._state = 2  # force a device read-back of the lower tiles
    assert np.array_equal(P.to_dense(tm), a)
    spd = O.spd_matrix(n, 2)
    tm = P.from_dense(spd, b)
    trace = tmp_path / "trace.csv"
    P.execute(P.gen_inversion(4, P.VariantConfig()), tm, trace_path=str(trace))
    rows = trace.read_text().strip().split("\n")
    assert rows[0] == "task_id,kind,indices,worker,start_ns,end_ns"
    assert len(rows) == 1 + 60
    for r in rows[1:]:
        tid, kind, idx, w, s, e = r.split(",")
        assert 0 <= int(s) <= int(e)


# ---------------------------------------------------------------- BASELINE config 4 (batched)
@pytest.mark.parametrize("nb", [256, 128])
def test_batched_inversion_vs_oracle(nb):
    rng = np.random.default_rng(4)
    batch, n = 24, 256
    g = rng.standard_normal((batch, n, n))
    a = g @ g.transpose(0, 2, 1) / n + np.eye(n)
    a = np.tril(a) + np.transpose(np.tril(a, -1), (0, 2, 1))
    x = P.invert_batched(a, nb)
    for k in range(0, batch, 5):
        ref = O.invert(a[k], nb)
        assert rel(x[k], ref) <= 1e-10 * np.linalg.cond(a[k])
        assert O.residual(a[k], x[k]) < 10


def test_batched_failure_reports_matrix():
    rng = np.random.default_rng(5)
    batch, n = 6, 128
    g = rng.standard_normal((batch, n, n))
    a = g @ g.transpose(0, 2, 1) / n + np.eye(n)
    a[3, 40, 40] = -2.0
    with pytest.raises(P.ExecutionError) as ei:
        P.invert_batched(a, 64)
    assert ei.value.matrix == 3
    assert isinstance(ei.value.cause, P.NotPositiveDefiniteError)
    assert ei.value.task.kind is P.KernelKind.POTRF


# ---------------------------------------------------------------- C4: fused per-matrix engine (csrc/batched.cu)
def _spd_batch(batch, n, seed, shift=1.0):
    g = np.random.default_rng(seed).standard_normal((batch, n, n))
    a = g @ g.transpose(0, 2, 1) / n + shift * np.eye(n)
    return np.tril(a) + np.transpose(np.tril(a, -1), (0, 2, 1))


@pytest.fixture(params=["cta", "pipe"])
def batch_engine(request):
    """Both fused engines (tinv_batch_small_engine): one block per matrix, and the
    pipelined persistent engine (even 64 <= n <= 256; other n fall back to cta)."""
    prev = _native.batch_engine(request.param)
    yield request.param
    _native.batch_engine(prev)


@pytest.mark.parametrize("n", [1, 2, 5, 33, 64, 65, 100, 128, 130, 191, 200, 255, 256])
def test_fused_batched_vs_oracle(n, batch_engine):
    """gen_inversion(1) per matrix fused in one CTA: parity with the oracle's
    POTRF -> TRTRI -> LAUUM of the single tile (odd n: synchronous loads;
    n % 64 != 0: identity-padded blocks)."""
    a = _spd_batch(7, n, 40 + n, 0.5)
    x = P.invert_batched(a, n, engine="fused")
    assert np.array_equal(x, np.transpose(x, (0, 2, 1)))  # exactly symmetric
    for k in range(a.shape[0]):
        ref = O.invert(a[k], n)
        assert rel(x[k], ref) <= 1e-10 * np.linalg.cond(a[k])
        assert O.residual(a[k], x[k]) < 10
    assert np.array_equal(P.invert_batched(a, n, engine="fused"), x)  # deterministic


def test_fused_batched_matches_dag_engine_and_device_api(batch_engine):
    import torch

    a = _spd_batch(300, 256, 7)
    xf = P.invert_batched(a, 256)  # auto -> fused
    xd = P.invert_batched(a, 256, engine="dag")
    assert rel(xf, xd) <= 1e-10 * max(np.linalg.cond(a[k]) for k in range(0, 300, 50))
    # device-pointer entry point, out of place and in place: same bits
    da = torch.from_numpy(a).cuda()
    dx = torch.empty_like(da)
    fail = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _native.batch_small_launch(da.data_ptr(), dx.data_ptr(), 300, 256, 256 * 256, st, fail.data_ptr())
    torch.cuda.synchronize()
    assert int(fail.item()) == -1
    assert np.array_equal(dx.cpu().numpy(), xf)
    _native.batch_small_launch(da.data_ptr(), da.data_ptr(), 300, 256, 256 * 256, st, fail.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(da.cpu().numpy(), xf)
    # pinned host buffers through the chunked pipeline (several chunks)
    big = np.concatenate([a] * 4)
    hb, hy = _pinned(big.shape), _pinned(big.shape)
    hb[...] = big
    P.invert_batched_host(hb, out=hy)
    assert np.array_equal(hy, np.concatenate([xf] * 4))


def test_fused_engines_agree():
    """The two fused engines run the same block algorithm (64x64 blocks, the
    same per-element summation order is NOT guaranteed): normwise agreement."""
    a = _spd_batch(150, 256, 11)
    prev = _native.batch_engine("cta")
    try:
        xc = P.invert_batched(a, 256)
        _native.batch_engine("pipe")
        xp = P.invert_batched(a, 256)
    finally:
        _native.batch_engine(prev)
    assert np.array_equal(xp, np.transpose(xp, (0, 2, 1)))
    for k in range(0, 150, 37):
        assert rel(xp[k], xc[k]) <= 1e-10 * np.linalg.cond(a[k])


@pytest.mark.parametrize("n,col", [(256, 10), (256, 200), (100, 70), (33, 0)])
def test_fused_batched_failure_reports_matrix_and_column(n, col, batch_engine):
    a = _spd_batch(9, n, 3)
    a[6, col, col] = -5.0
    a[4, col, col] = -5.0  # the lowest failing matrix is reported
    with pytest.raises(O.NotPositiveDefinite) as eo:
        O.potrf(np.tril(a[4]))
    with pytest.raises(P.ExecutionError) as ei:
        P.invert_batched(a, n)
    assert ei.value.matrix == 4
    assert isinstance(ei.value.cause, P.NotPositiveDefiniteError)
    assert ei.value.cause.index == eo.value.index
    assert ei.value.task.kind is P.KernelKind.POTRF
    a[4, col, col] = np.nan
    with pytest.raises(P.ExecutionError) as ei:
        P.invert_batched_host(a, out=np.empty_like(a))
    assert ei.value.matrix == 4 and ei.value.cause.index == eo.value.index


# ---------------------------------------------------------------- multi-GPU distribution (loopback)
@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (2, 4)])
def test_distributed_loopback_bitwise(grid):
    from paper_1002_4057_b200.distributed import execute_distributed
    n, b = 1024, 128
    a = O.spd_matrix(n, 6, 0.5)
    for cfg in (P.VariantConfig(P.Placement.OUT_OF_PLACE), P.VariantConfig(P.Placement.IN_PLACE, "UUU", False)):
        s = P.gen_inversion(n // b, cfg)
        ref = P.from_dense(a, b)
        P.execute(s, ref)
        tm = P.from_dense(a, b)
        d = execute_distributed(s, tm, grid)
        assert np.array_equal(P.to_dense(tm), P.to_dense(ref))
        assert d.stats(b)["transfers"] > 0


@pytest.mark.parametrize("grid,partition", [((1, 2), False), ((2, 2), False), ((1, 2), True), ((2, 2), True),
                                            ((2, 4), True)])
def test_distributed_separate_stores_concurrent_ranks(grid, partition):
    """The multi-process runtime's data path with every rank in this process:
    one store and one transfer plan per rank (what MultiGPU builds), the ranks'
    persistent executors running concurrently on disjoint SM shares, SENDs
    writing into the OTHER stores and inboxes (tinv_peer_attach). partition:
    each store holds only its rank's tiles. Bitwise equal to execute()."""
    from paper_1002_4057_b200.distributed import execute_ranks_local
    n, b = 1024, 128
    a = O.spd_matrix(n, 8, 0.5)
    for cfg in (P.VariantConfig(P.Placement.OUT_OF_PLACE), P.VariantConfig(P.Placement.IN_PLACE, "UUU", False)):
        s = P.gen_inversion(n // b, cfg)
        ref = P.from_dense(a, b)
        P.execute(s, ref)
        tm = P.from_dense(a, b)
        d, ms, store = execute_ranks_local(s, tm, grid, partition=partition)
        assert np.array_equal(P.to_dense(tm), P.to_dense(ref))
        assert len(ms) == grid[0] * grid[1] and d.stats(b)["transfers"] > 0
        if partition:
            full = _native.Context(n, b).store_bytes()
            assert max(store) < full  # a rank keeps its own tiles, not the whole matrix


def test_partitioned_store_transfers_only_owned_tiles():
    """tinv_create_owned: put_dense / get_dense move this rank's tiles only (one
    2D copy per tile); other ranks' tiles of the host buffer stay untouched,
    and plans touching them are rejected."""
    from paper_1002_4057_b200.distributed import owned_tiles
    n, b, grid = 640, 128, (2, 2)
    t = n // b
    a = O.spd_matrix(n, 3, 0.5)
    for r in range(4):
        own = owned_tiles(t, grid, r)
        ctx = _native.Context.owned(n, b, own)
        assert ctx.store_bytes() < _native.Context(n, b).store_bytes()
        ctx.put_dense(a)
        out = np.full((n, n), 7.0)
        ctx.get_dense(out, _native.DENSE_LOWER)
        for i in range(t):
            for j in range(t):
                blk = out[i * b:(i + 1) * b, j * b:(j + 1) * b]
                if j <= i and own[i, j]:
                    assert np.array_equal(blk, a[i * b:(i + 1) * b, j * b:(j + 1) * b])
                else:
                    assert (blk == 7.0).all()
        with pytest.raises(_native.NativeError):
            ctx.get_dense(out, _native.DENSE_SYMMETRIZE)
        s = P.gen_inversion(t, P.VariantConfig())  # the whole stream touches every tile
        plan = _native.Plan(ctx, s.table(), t, np.zeros(0, np.int64))
        assert plan.rc != _native.OK and "another rank" in plan.msg
        ctx.close()


@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (2, 4)])
def test_distributed_device_transport_bitwise(grid):
    # SEND (CTA copy into the receiver's pool + system-scope inbox flag) and
    # RECV (completed by the inbox poller), every rank in one launch
    from paper_1002_4057_b200.distributed import execute_distributed
    n, b = 1024, 128
    a = O.spd_matrix(n, 7, 0.5)
    s = P.gen_inversion(n // b, P.VariantConfig(P.Placement.OUT_OF_PLACE))
    ref = P.from_dense(a, b)
    P.execute(s, ref)
    tm = P.from_dense(a, b)
    execute_distributed(s, tm, grid, transport="device")
    assert np.array_equal(P.to_dense(tm), P.to_dense(ref))


@pytest.mark.parametrize("grid", [(1, 2), (1, 3), (2, 2), (2, 4)])
def test_distributed_ranks_in_one_launch_bitwise(grid):
    # every rank on its own group of nsm / P*Q CTAs with its own priority
    # queues (tinv_plan_create_ranks): the multi-GPU schedule in one launch
    from paper_1002_4057_b200.distributed import execute_distributed
    n, b = 1280, 128
    a = O.spd_matrix(n, 12, 0.5)
    for cfg in (P.VariantConfig(P.Placement.OUT_OF_PLACE), P.VariantConfig(P.Placement.IN_PLACE, "UDU", True)):
        s = P.gen_inversion(n // b, cfg)
        ref = P.from_dense(a, b)
        P.execute(s, ref)
        tm = P.from_dense(a, b)
        d = execute_distributed(s, tm, grid, transport="ranks")
        assert np.array_equal(P.to_dense(tm), P.to_dense(ref))
        run = d.last_run
        world = grid[0] * grid[1]
        assert len(run["cta_idle_ns"]) % world == 0 and set(run["cta_rank"].tolist()) == set(range(world))
        assert (run["cta_idle_ns"] >= 0).all() and (run["cta_idle_ns"] <= run["kernel_ms"] * 1e6 * 1.01).all()


# ---------------------------------------------------------------- streamed host I/O (tinv_plan_exec_host)
def _pinned(shape):
    import torch

    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()


@pytest.mark.parametrize("n,b,placement,pipelined", [(1536, 128, "out", True), (1000, 200, "in", True),
                                                      (1152, 384, "out", False), (256, 256, "in", True)])
def test_streamed_host_io_bitwise(n, b, placement, pipelined):
    a = O.spd_matrix(n, 7, 0.5)
    cfg = P.VariantConfig(P.Placement(placement), "UDU", pipelined)
    ref = P.invert(a, b, cfg)
    ha, hx = _pinned(a.shape), _pinned(a.shape)
    ha[...] = a
    for _ in range(2):  # second call: cached plan and store
        hx.fill(np.nan)
        P.invert_host(ha, b, cfg, out=hx)
        assert np.array_equal(hx, ref)
    # pageable output: staged fallback, same bits
    assert np.array_equal(P.invert_host(a, b, cfg), ref)
    P.clear_plan_cache()


def test_streamed_lower_mode_and_batched():
    n, b = 640, 128
    a = O.spd_matrix(n, 8, 0.5)
    t = n // b
    s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE))
    ctx = _native.Context(n, b)
    ctx.put_dense(a)
    plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
    assert plan.run()[0] == 0
    lower = np.full((n, n), np.nan)
    ctx.get_dense(lower, _native.DENSE_LOWER)
    plan.close()
    sp = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), _native.STREAM_IO)
    ha, hx = _pinned((n, n)), _pinned((n, n))
    ha[...] = a
    hx.fill(np.nan)
    rc, err, ms = sp.run_host(ha.ctypes.data, n, hx.ctypes.data, n, _native.DENSE_LOWER)
    assert rc == 0, sp.msg
    assert np.array_equal(np.isnan(hx), np.isnan(lower))  # upper tiles untouched
    assert np.array_equal(np.nan_to_num(hx), np.nan_to_num(lower))
    assert sp.run()[0] == _native.ERR_BAD_ARG  # a STREAM_IO plan needs host buffers
    sp.close()
    # a staged run on the same store after the streamed run re-homed its tiles
    # (column-major home slots, api.cu plan_exec_impl): same bits
    ctx.put_dense(a)
    plan2 = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64))
    assert plan2.run()[0] == 0
    again = np.full((n, n), np.nan)
    ctx.get_dense(again, _native.DENSE_LOWER)
    plan2.close()
    assert np.array_equal(np.nan_to_num(again), np.nan_to_num(lower))
    ctx.close()
    rng = np.random.default_rng(4)
    g = rng.standard_normal((40, 256, 256))
    ab = g @ g.transpose(0, 2, 1) / 256 + np.eye(256)
    ab = np.tril(ab) + np.transpose(np.tril(ab, -1), (0, 2, 1))
    for nb in (256, 128):
        ref = P.invert_batched(ab, nb)
        hb, hy = _pinned(ab.shape), _pinned(ab.shape)
        hb[...] = ab
        P.invert_batched_host(hb, nb, out=hy)
        assert np.array_equal(hy, ref)
    P.clear_plan_cache()


def test_streamed_failure_reports_task():
    a = O.spd_matrix(512, 9, 0.5)
    a[300, 300] = -50.0  # not SPD: POTRF of diagonal tile 2 (b=128) fails
    ha, hx = _pinned(a.shape), _pinned(a.shape)
    ha[...] = a
    with pytest.raises(P.ExecutionError) as ei:
        P.invert_host(ha, 128, out=hx)
    with pytest.raises(P.ExecutionError) as ej:
        P.invert(a, 128)
    assert str(ei.value.task) == str(ej.value.task)
    assert ei.value.cause.index == ej.value.cause.index
    P.clear_plan_cache()


_SERIALISED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1002_4057_b200 as P
from oracle import tileinv_oracle as O
n, b = 768, 128
a = O.spd_matrix(n, 11, 0.5)
cfg = P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True)
ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
ha[...] = a
P.invert_host(ha, b, cfg, out=hx)
ref = P.invert(a, b, cfg)
assert np.array_equal(hx, ref), "streamed != staged"
print("SERIALISED_OK")
"""


@pytest.mark.parametrize("env", [{"CUDA_LAUNCH_BLOCKING": "1"}, {"CUDA_DEVICE_MAX_CONNECTIONS": "1"}])
def test_streamed_host_path_under_serialised_launches(env):
    """The streamed path must make forward progress when kernel launches are
    serialised (a profiler's replay, CUDA_LAUNCH_BLOCKING, one hardware
    connection): the persistent executor spins on arrival flags, so the
    arrival copies are enqueued before it launches (api.cu plan_exec_impl)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _SERIALISED_SCRIPT.format(root=root)], env=e, capture_output=True,
                       text=True, timeout=240)
    assert r.returncode == 0 and "SERIALISED_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("n,b,placement,loops", [(1280, 128, "out", "UDU"), (1024, 256, "out", "DDU"),
                                                 (1000, 200, "in", "UDU"), (1536, 128, "out", "UUU")])
def test_share_slots_bitwise_and_smaller(n, b, placement, loops):
    """Memory-constrained renaming (TINV_SHARE_SLOTS): working tiles share
    slots by live range, reuse ordered by added edges -- same bits, smaller
    store (out-of-place: C reuses B's slots)."""
    a = O.spd_matrix(n, 13, 0.5)
    cfg = P.VariantConfig(P.Placement(placement), loops, True)
    t = n // b
    s = P.gen_inversion(t, cfg)
    outs, sizes = [], []
    for fl in (0, _native.SHARE_SLOTS):
        ctx = _native.Context(n, b)
        ctx.put_dense(a)
        plan = _native.Plan(ctx, s.table(), t, np.array(sorted(s.barriers), np.int64), fl)
        assert plan.run()[0] == 0, plan.msg
        x = np.zeros((n, n))
        ctx.get_dense(x, _native.DENSE_SYMMETRIZE)
        sizes.append(ctx.store_bytes())
        plan.close()
        ctx.close()
        outs.append(x)
    assert np.array_equal(outs[0], outs[1])
    assert O.normwise_diff(outs[1], O.invert(a, b, loops, placement == "out", True)) <= 1e-10 * np.linalg.cond(a)
    if placement == "out":
        assert sizes[1] < sizes[0]
    assert np.array_equal(P.invert(a, b, cfg, share_slots=True), outs[0])


@pytest.mark.parametrize("grid", [(1, 2), (2, 2)])
def test_multi_process_ipc_path_on_one_gpu(grid):
    """The multi-PROCESS data path (`execute_multi_gpu`: CUDA-IPC mapped
    partitioned stores, receive bases, system-scope inbox flags, owned-tile
    gather), two / four ranks as separate processes and CUDA contexts sharing
    cuda:0 (gloo control plane; the driver time-slices the executors), bitwise
    against one process running scheduler.py:261-351's `execute`."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "two_proc_one_gpu.py"), "512", "128",
                            str(grid[0]), str(grid[1])], capture_output=True, text=True, timeout=400)
    except subprocess.TimeoutExpired:  # the ranks only advance by driver time slices: slow is not wrong
        pytest.skip("time-sliced ranks did not finish in 400 s")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "bitwise equal to one process: True" in r.stdout


def test_bench_multi_rank_path_on_one_gpu():
    """bench.py's N > 1 path under the driver's torchrun launch line, two ranks
    as separate processes on cuda:0 (TINV_BENCH_ONE_GPU=1: gloo control plane,
    time-sliced executors -- a functional check, the numbers mean nothing)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TINV_BENCH_ONE_GPU="1")
    import socket
    with socket.socket() as sk:  # a free rendezvous port
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    try:
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                            "--master-addr", "127.0.0.1", "--master-port", str(port),
                            os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "c1", "--steps", "2",
                            "--warmup", "3", "--no-cpu"], capture_output=True, text=True, timeout=600, env=env,
                           cwd=root)
    except subprocess.TimeoutExpired:
        pytest.skip("time-sliced ranks did not finish in 600 s")
    assert r.returncode == 0, r.stdout[-1500:] + r.stderr[-1500:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["transfers"] > 0 and d["residual"] < 10 and d["symmetry_err"] == 0.0
    assert d["e2e"]["value"] > 0
