"""Host-side logic of the product package, CPU only: the C-ABI library loads
and exports every header symbol; native stream generation, the native hazard
scoreboard and the analysis API reproduce the reference (golden fixtures from
the live reference, tests/golden/streams.json) and the oracle."""

import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_1002_4057_b200 as P
from paper_1002_4057_b200 import _native
from oracle import tileinv_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def streams():
    with open(os.path.join(GOLD, "streams.json")) as fh:
        return json.load(fh)


def test_library_exports_every_header_symbol():
    L = _native.lib()
    with open(os.path.join(ROOT, "include", "tileinv_b200.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"\b(tinv_[a-z_]+)\s*\(", hdr))
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.tinv_abi_version() == 1


def _variant(key):
    t, pl, loops, pipe = key.split("_")
    return int(t[1:]), P.VariantConfig(P.Placement(pl), loops, pipe == "1")


def test_full_streams_match_reference(streams):
    for key, g in streams["full"].items():
        t, cfg = _variant(key)
        s = P.gen_inversion(t, cfg)
        txt = P.format_stream(s)
        assert len(s) == g["ntasks"], key
        assert hashlib.sha256(txt.encode()).hexdigest() == g["sha"], key
        if g["text"] is not None:
            assert txt == g["text"]


def test_step_streams_match_reference(streams):
    for key, g in streams["step"].items():
        parts = key.split("_")
        t, step, d = int(parts[0][1:]), int(parts[1][1:]), parts[-1]
        pl = P.Placement(parts[2]) if len(parts) == 4 else P.Placement.IN_PLACE
        s = {1: lambda: P.gen_step1(t, d), 2: lambda: P.gen_step2(t, d, pl), 3: lambda: P.gen_step3(t, d, pl)}[step]()
        assert hashlib.sha256(P.format_stream(s).encode()).hexdigest() == g["sha"], key


def test_native_dag_matches_reference(streams):
    for key, g in streams["step"].items():
        if g["edges"] is None:
            continue
        parts = key.split("_")
        t, step, d = int(parts[0][1:]), int(parts[1][1:]), parts[-1]
        pl = P.Placement(parts[2]) if len(parts) == 4 else P.Placement.IN_PLACE
        s = {1: lambda: P.gen_step1(t, d), 2: lambda: P.gen_step2(t, d, pl), 3: lambda: P.gen_step3(t, d, pl)}[step]()
        dag = P.build_dag(s)
        got = sorted([e.src, e.dst, e.kind.value if e.kind else "BAR"] for e in dag.edges)
        assert got == g["edges"], key
    for key, g in streams["full"].items():
        t, cfg = _variant(key)
        dag = P.build_dag(P.gen_inversion(t, cfg))
        assert len(dag.edges) == g["nedges"], key
        rep = P.critical_path(dag)
        assert rep.critical_path == g["cp"], key
        assert rep.copy_inclusive_path == g["cp_copies"], key
        cen = P.hazard_census(dag)
        for kind, cats in g["census"].items():
            for cat, cnt in cats.items():
                assert cen[P.HazardKind(kind)][cat] == cnt, (key, kind, cat)


@pytest.mark.parametrize("t", [2, 5, 9])
def test_native_dag_matches_oracle_edges(t):
    for pl in P.Placement:
        for loops in ("UDU", "DUD"):
            for pipe in (True, False):
                s = P.gen_inversion(t, P.VariantConfig(pl, loops, pipe))
                so = O.gen_stream(t, (1, 2, 3), loops, pl is P.Placement.OUT_OF_PLACE, pipe)
                src, dst, kind = _native.dag_edges(s.table(), sorted(s.barriers))
                names = ["RAW", "WAR", "WAW", "BAR"]
                got = sorted(zip(src.tolist(), dst.tolist(), [names[k] for k in kind.tolist()]))
                assert got == sorted(O.build_edges(so))


def test_table1_formulas():
    # PAPER Table 1 holds exactly for t=2..8; the pipelined rows
    # of the reference do not (SURVEY.md finding 6) -- same here.
    rows = P.formula_table(range(2, 9))
    bad = {r.variant for r in rows if not r.match}
    assert bad == {"full/in/pipelined", "full/out/pipelined"}
    assert P.formula_csv(rows).startswith("variant,t,measured,formula,match\n")


def test_spec_structural_examples():
    # SPEC.md:242-244, 251-253, 260-262, 269-271
    assert [str(x) for x in P.gen_step1(1).tasks] == ["POTRF(0)"]
    assert len(P.gen_step1(4).tasks) == 20
    assert [str(x) for x in P.gen_step2(2, "D").tasks] == ["TRTRI(1)", "TRTRI(0)", "TRMM_LEFT(1,0)",
                                                          "TRMM_RIGHT_NEG(1,0)"]
    assert sum(1 for x in P.gen_step2(4).tasks if x.kind is P.KernelKind.GEMM) == 4
    assert [str(x) for x in P.gen_step3(1).tasks] == ["LAUUM(0)"]
    assert len(P.gen_inversion(4, P.VariantConfig()).tasks) == 60
    s = P.gen_inversion(4, P.VariantConfig(P.Placement.OUT_OF_PLACE))
    assert sum(x.is_copy for x in s.tasks) == 20 and len(s.tasks) == 80
    # WAR SYRK(0,1) -> TRMM(1,0) in step 3 in-place t=2
    dag = P.build_dag(P.gen_step3(2, "U"))
    war = [(e.src, e.dst) for e in dag.edges if e.kind is P.HazardKind.WAR]
    names = {(str(dag.tasks[u]), str(dag.tasks[v])) for u, v in war}
    assert ("SYRK_ADD_T(0,1)", "TRMM_LEFT_T(1,0)") in names
    # zero WAR among kernel tasks out-of-place
    for t in range(2, 7):
        for s in (P.gen_step2(t, "D", P.Placement.OUT_OF_PLACE), P.gen_step3(t, "U", P.Placement.OUT_OF_PLACE)):
            assert P.hazard_census(P.build_dag(s))[P.HazardKind.WAR]["intra_step"] == 0
    # SPEC.md:336-338 ready set
    d1 = P.build_dag(P.gen_step1(2))
    assert P.ready_set(d1, set()) == {0}
    assert {str(d1.tasks[i]) for i in P.ready_set(d1, {0})} == {"TRSM(1,0)"}
    assert P.weak_components(P.build_dag(P.gen_step3(4, "U", P.Placement.OUT_OF_PLACE))) > 1


def test_stream_encoding_roundtrip():
    for cfg in (P.VariantConfig(), P.VariantConfig(P.Placement.OUT_OF_PLACE, "DUD", False)):
        s = P.gen_inversion(5, cfg)
        native = s.table()
        from paper_1002_4057_b200.taskgen import encode_tasks
        assert np.array_equal(encode_tasks(s.tasks), native)
        user = P.TaskStream(list(s.tasks), set(s.barriers), s.t, s.steps, s.placement, s.loops)
        assert user == s
        assert np.array_equal(user.table(), native)


def test_api_validation_without_gpu():
    with pytest.raises(P.InvalidSizeError):
        P.from_dense(np.eye(6), 4)
    with pytest.raises(ValueError):
        P.from_dense(np.full((2, 2), np.nan), 1)
    with pytest.raises(ValueError):
        P.VariantConfig(loops="UXU")
    with pytest.raises(ValueError):
        P.VariantConfig(workers=0)
    tm = P.from_dense(np.eye(4), 2)
    with pytest.raises(ValueError):
        P.execute(P.gen_step1(2), tm, workers=0)
    with pytest.raises(P.InvalidStreamError):
        P.execute(P.gen_step1(3), tm)
    assert P.to_dense(tm).tolist() == np.eye(4).tolist()
    assert [str(x) for x in tm.lower_ids()] == ["A[0,0]", "A[1,0]", "A[1,1]"]
    with pytest.raises(P.ShapeMismatchError):
        P.max_abs_diff(np.eye(2), np.eye(3))


def test_no_cpu_fallback_without_device():
    if _native.device_count() > 0:
        pytest.skip("a B200 is present")
    tm = P.from_dense(np.eye(4) * 4.0, 2)
    with pytest.raises(_native.NativeError):
        P.execute(P.gen_inversion(2, P.VariantConfig()), tm)


def test_batched_validation():
    with pytest.raises(P.InvalidSizeError):
        P.invert_batched(np.zeros((2, 4, 5)), 2)
    with pytest.raises(P.InvalidSizeError):
        P.invert_batched(np.zeros((2, 6, 6)), 4)
    with pytest.raises(ValueError):
        P.invert_batched(np.full((1, 2, 2), np.inf), 2)


def test_invert_host_validation():
    a = np.eye(8) * 2.0
    with pytest.raises(ValueError):
        P.invert_host(a, 4, out=a)  # in-place would race the streamed copies
    with pytest.raises(ValueError):
        P.invert_host(a, 4, out=np.empty((8, 8), dtype=np.float32))
    with pytest.raises(P.InvalidSizeError):
        P.invert_host(np.eye(6), 4)
    with pytest.raises(P.InvalidSizeError):
        P.invert_batched_host(np.eye(4), 2)


def test_fused_batched_engine_selection_and_abi_validation():
    """Routing of invert_batched's engines (host logic) and the fused C-ABI
    entry points' argument checks (they fail before touching a device)."""
    from paper_1002_4057_b200.inversion import _fused_ok

    assert _fused_ok(256, 256, "auto") and _fused_ok(1, 1, "fused")
    assert not _fused_ok(256, 128, "auto") and not _fused_ok(512, 512, "auto")
    assert not _fused_ok(256, 256, "dag")
    with pytest.raises(ValueError):
        _fused_ok(256, 128, "fused")  # the fused engine needs nb == n <= 256
    with pytest.raises(ValueError):
        _fused_ok(256, 256, "gpu")
    with pytest.raises(ValueError):
        P.invert_batched(np.stack([np.eye(4)] * 2), 2, engine="fused")
    L = _native.lib()
    fake = ctypes.c_void_p(16)
    assert L.tinv_batch_small_launch(None, None, 1, 4, 16, None, None) == _native.ERR_BAD_ARG
    assert L.tinv_batch_small_launch(fake, fake, 1, 300, 300 * 300, None, fake) == _native.ERR_BAD_ARG
    assert L.tinv_batch_small_launch(fake, fake, 1, 8, 10, None, fake) == _native.ERR_BAD_ARG  # stride < n*n
    fm, fi = ctypes.c_int64(0), ctypes.c_int64(0)
    assert L.tinv_batch_small_host(fake, fake, 1, 257, 0, ctypes.byref(fm), ctypes.byref(fi), None) == \
        _native.ERR_BAD_ARG
    assert (fm.value, fi.value) == (-1, -1)
    # engine selection is host state (no device needed)
    prev = _native.batch_engine("pipe")
    assert _native.batch_engine() == "pipe"
    assert _native.batch_engine("cta") == "pipe"
    assert L.tinv_batch_small_engine(7) == 0 and _native.batch_engine() == "cta"  # unknown values only query
    _native.batch_engine(prev)


def test_multi_rank_abi_validation_host_only():
    """The multi-rank entry points reject bad arguments without a device:
    tinv_peer_attach / tinv_set_sms / tinv_create_owned / tinv_recv_base /
    tinv_ipc_recv_bases (include/tileinv_b200.h)."""
    import ctypes
    L = _native.lib()
    assert L.tinv_set_sms(None, 4) == _native.ERR_BAD_ARG
    assert L.tinv_peer_attach(None, 0, 1, None) == _native.ERR_BAD_ARG
    assert L.tinv_ipc_recv_bases(None, 1, None) == _native.ERR_BAD_ARG
    assert L.tinv_recv_base(None, None) == _native.ERR_BAD_ARG
    h = ctypes.c_void_p()
    assert L.tinv_create_owned(ctypes.byref(h), 256, 128, 0, None) == _native.ERR_BAD_ARG  # null mask
    # with a mask but no device: no store is created
    own = np.ones((2, 2), np.int32)
    rc = L.tinv_create_owned(ctypes.byref(h), 256, 128, 0, own.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    assert rc == _native.ERR_NO_DEVICE and not h.value


def test_owned_tiles_partition_the_lower_tiles():
    """distributed.owned_tiles: the 2D block-cyclic ownership masks of the
    ranks of a grid cover every lower tile exactly once."""
    from paper_1002_4057_b200.distributed import owned_tiles
    for grid in ((1, 1), (1, 2), (2, 2), (2, 4)):
        t = 9
        tot = sum(owned_tiles(t, grid, r) for r in range(grid[0] * grid[1]))
        assert np.array_equal(tot, np.tril(np.ones((t, t), np.int32)))


def test_schedule_model_host_only():
    """csrc/model.cu: the executor's schedule simulated on the host (no GPU):
    deadlock-free on single-GPU and transfer plans, busy SM-time independent of
    the SM count, makespan bounded below by busy/SMs and by the unlimited-SM run."""
    from paper_1002_4057_b200.distributed import distribute, transfer_plan
    n, b = 2048, 256
    t = n // b
    s = P.gen_inversion(t, P.VariantConfig(P.Placement.OUT_OF_PLACE, "UDU", True))
    mk, busy = _native.model_run(n, b, s.table(), t, sorted(s.barriers), sms_per_rank=148)
    mk4, busy4 = _native.model_run(n, b, s.table(), t, sorted(s.barriers), sms_per_rank=4)
    cp, _ = _native.model_run(n, b, s.table(), t, sorted(s.barriers), sms_per_rank=100000)
    assert abs(busy[0] - busy4[0]) < 1e-6 * busy[0]
    assert mk4 >= busy4[0] / 4 - 1e-6 and mk >= cp - 1e-6 and mk4 >= mk - 1e-6
    for grid in ((1, 2), (2, 2), (2, 4)):
        d = distribute(s, grid)
        table, aux, nrecv, _, who = transfer_plan(d, -1, with_ranks=True)
        w = grid[0] * grid[1]
        mkd, bd, crit = _native.model_run(n, b, table, t, aux=aux, nrecv=nrecv, rank_of=who, nranks=w,
                                          sms_per_rank=148 // w, with_crit=True)
        assert len(bd) == w and (bd > 0).all() and mkd > 0
        assert abs(sum(crit.values()) - mkd) < 1e-6 * mkd  # the critical chain spans the run


def test_rank_plan_rejects_bad_ranks():
    with pytest.raises(_native.NativeError):
        s = P.gen_inversion(4, P.VariantConfig())
        _native.model_run(512, 128, s.table(), 4, sorted(s.barriers), nranks=9, rank_of=np.zeros(len(s), np.int32))
