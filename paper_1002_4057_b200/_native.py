"""ctypes binding of libtileinv_b200.so (include/tileinv_b200.h).

The library is the product: every numeric operation of the package runs
through it on the B200. There is no CPU fallback -- if the library is missing
or no sm_100 device is present, calls raise.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TINV_LIB") or os.path.join(_PKG, "libtileinv_b200.so")

TASK_FIELDS = 16
OK, ERR_NOT_SPD, ERR_SINGULAR, ERR_BAD_ARG, ERR_CUDA, ERR_STREAM, ERR_NO_DEVICE, ERR_INTERNAL = range(8)
SERIAL, TRACE, KEEP_ON_FAILURE, STREAM_IO, SHARE_SLOTS = 1, 2, 4, 8, 16
DENSE_LOWER, DENSE_SYMMETRIZE = 0, 1

# every symbol include/tileinv_b200.h declares
EXPORTS = (
    "tinv_abi_version", "tinv_device_count", "tinv_last_error", "tinv_create", "tinv_create_batch", "tinv_destroy",
    "tinv_shape", "tinv_store_bytes", "tinv_set_stream", "tinv_put_dense", "tinv_get_dense", "tinv_put_dense_device", "tinv_get_dense_device",
    "tinv_put_tile", "tinv_get_tile", "tinv_gen_stream", "tinv_dag_edges", "tinv_dag_paths", "tinv_dist_stream", "tinv_plan_create",
    "tinv_plan_create_xfer", "tinv_plan_create_ranks", "tinv_plan_cta_idle", "tinv_model_run", "tinv_ipc_export", "tinv_ipc_open", "tinv_ipc_reset", "tinv_peer_attach", "tinv_set_sms", "tinv_create_owned", "tinv_recv_base", "tinv_ipc_recv_bases", "tinv_plan_exec",
    "tinv_plan_exec_host", "tinv_plan_destroy", "tinv_plan_stats", "tinv_plan_trace", "tinv_run",
    "tinv_batch_small_launch", "tinv_batch_small_host", "tinv_batch_small_engine",
)
BATCH_SMALL_MAX_N = 256  # tinv_batch_small_*: 1 <= n <= 256


class TinvErr(ctypes.Structure):
    _fields_ = [("task_id", ctypes.c_int32), ("kind", ctypes.c_int32), ("code", ctypes.c_int32),
                ("index", ctypes.c_int32)]


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"libtileinv_b200 error {code}: {msg}")


_lib = None

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_DP = ctypes.POINTER(ctypes.c_double)
_I32P = ctypes.POINTER(ctypes.c_int32)
_I64P = ctypes.POINTER(ctypes.c_int64)


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                           "(nvcc, sm_100a); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "tinv_abi_version": ([], ctypes.c_int),
        "tinv_device_count": ([], ctypes.c_int),
        "tinv_last_error": ([_P], ctypes.c_char_p),
        "tinv_create": ([ctypes.POINTER(_P), _I64, _I64, ctypes.c_int], ctypes.c_int),
        "tinv_create_batch": ([ctypes.POINTER(_P), _I64, _I64, _I64, ctypes.c_int], ctypes.c_int),
        "tinv_destroy": ([_P], ctypes.c_int),
        "tinv_shape": ([_P, _I64P, _I64P, _I64P, _I64P], ctypes.c_int),
        "tinv_store_bytes": ([_P, _I64P], ctypes.c_int),
        "tinv_set_stream": ([_P, _P], ctypes.c_int),
        "tinv_put_dense": ([_P, _DP, _I64], ctypes.c_int),
        "tinv_get_dense": ([_P, _DP, _I64, ctypes.c_int], ctypes.c_int),
        "tinv_put_dense_device": ([_P, _P, _I64], ctypes.c_int),
        "tinv_get_dense_device": ([_P, _P, _I64, ctypes.c_int], ctypes.c_int),
        "tinv_put_tile": ([_P, _I64, _I64, _DP], ctypes.c_int),
        "tinv_get_tile": ([_P, _I64, _I64, _DP], ctypes.c_int),
        "tinv_gen_stream": ([_I32, _I32, ctypes.c_char_p, _I32, _I32, _I32P, _I64, _I64P, _I64P, _I64, _I64P],
                            ctypes.c_int),
        "tinv_dag_edges": ([_I32P, _I64, _I64P, _I64, _I32P, _I32P, ctypes.POINTER(ctypes.c_int8), _I64, _I64P],
                           ctypes.c_int),
        "tinv_dag_paths": ([_I32P, _I64, _I64P, _I64, _DP, _I32, _DP, _I32P, _I32P, _I64P], ctypes.c_int),
        "tinv_dist_stream": ([_I32P, _I64, _I32, _I32, _I32, _I32P, _I64, _I64P, _I32P, _I32P, _I32P], ctypes.c_int),
        "tinv_plan_create": ([_P, _I32P, _I64, _I32, _I64P, _I64, _U32, ctypes.POINTER(_P),
                              ctypes.POINTER(TinvErr)], ctypes.c_int),
        "tinv_plan_create_xfer": ([_P, _I32P, _I64, _I32, _I32P, _I64, _U32, ctypes.POINTER(_P),
                                   ctypes.POINTER(TinvErr)], ctypes.c_int),
        "tinv_plan_create_ranks": ([_P, _I32P, _I64, _I32, _I32P, _I64, _I32P, _I32, _U32, ctypes.POINTER(_P),
                                    ctypes.POINTER(TinvErr)], ctypes.c_int),
        "tinv_plan_cta_idle": ([_P, _I64P, _I32P, _I64, _I64P], ctypes.c_int),
        "tinv_model_run": ([_I64, _I64, _I32P, _I64, _I32, _I64P, _I64, _I32P, _I64, _I32P, _I32, _I32, _U32, _DP, _DP,
                            _DP],
                           ctypes.c_int),
        "tinv_ipc_export": ([_P, _P, ctypes.c_char_p, ctypes.c_char_p], ctypes.c_int),
        "tinv_ipc_open": ([_P, _I32, _I32, ctypes.c_char_p, ctypes.c_char_p], ctypes.c_int),
        "tinv_ipc_reset": ([_P], ctypes.c_int),
        "tinv_peer_attach": ([_P, _I32, _I32, ctypes.POINTER(_P)], ctypes.c_int),
        "tinv_set_sms": ([_P, _I32], ctypes.c_int),
        "tinv_create_owned": ([ctypes.POINTER(_P), _I64, _I64, ctypes.c_int, _I32P], ctypes.c_int),
        "tinv_recv_base": ([_P, _I32P], ctypes.c_int),
        "tinv_ipc_recv_bases": ([_P, _I32, _I32P], ctypes.c_int),
        "tinv_plan_exec": ([_P, ctypes.POINTER(TinvErr), ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "tinv_plan_exec_host": ([_P, _P, _I64, _P, _I64, ctypes.c_int, ctypes.POINTER(TinvErr),
                                 ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "tinv_plan_destroy": ([_P], ctypes.c_int),
        "tinv_plan_stats": ([_P, _I64P, _I64P, _I64P], ctypes.c_int),
        "tinv_plan_trace": ([_P, _I64P, _I64P, _I32P, _I64], ctypes.c_int),
        "tinv_run": ([_P, _I32P, _I64, _I32, _I64P, _I64, _U32, ctypes.POINTER(TinvErr)], ctypes.c_int),
        "tinv_batch_small_launch": ([_P, _P, _I64, _I64, _I64, _P, _P], ctypes.c_int),
        "tinv_batch_small_host": ([_P, _P, _I64, _I64, ctypes.c_int, _I64P, _I64P, ctypes.POINTER(ctypes.c_double)],
                                  ctypes.c_int),
        "tinv_batch_small_engine": ([ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.tinv_abi_version() != 1:
        raise RuntimeError("libtileinv_b200.so ABI mismatch")
    _lib = L
    return L


def _dp(a):
    return a.ctypes.data_as(_DP)


def _ip(a):
    return a.ctypes.data_as(_I32P) if a is not None else None


def _lp(a):
    return a.ctypes.data_as(_I64P) if a is not None and len(a) else None


def last_error(ctx=None):
    m = lib().tinv_last_error(ctx)
    return m.decode() if m else ""


def check(rc, ctx=None):
    if rc != OK:
        raise NativeError(rc, last_error(ctx))


def device_count():
    return lib().tinv_device_count()


def batch_small_launch(a_ptr, x_ptr, batch, n, stride, stream_ptr, fail_ptr):
    """Asynchronous fused batched inversion on device buffers (tinv_batch_small_launch)."""
    check(lib().tinv_batch_small_launch(a_ptr, x_ptr, batch, n, stride, stream_ptr, fail_ptr))


BATCH_ENGINES = {"cta": 0, "pipe": 1}


def batch_engine(name=None):
    """Select the fused batched engine ("cta" | "pipe", tinv_batch_small_engine);
    returns the previous one. None only queries."""
    prev = lib().tinv_batch_small_engine(-1 if name is None else BATCH_ENGINES[name])
    return {v: k for k, v in BATCH_ENGINES.items()}[prev]


def batch_small_host(a_ptr, x_ptr, batch, n, device=0):
    """Blocking fused batched inversion of host buffers; returns (rc, fail_matrix, fail_index, ms)."""
    fm, fi, ms = ctypes.c_int64(-1), ctypes.c_int64(-1), ctypes.c_double(0.0)
    rc = lib().tinv_batch_small_host(a_ptr, x_ptr, batch, n, device, ctypes.byref(fm), ctypes.byref(fi),
                                     ctypes.byref(ms))
    if rc not in (OK, ERR_NOT_SPD):
        check(rc)
    return rc, fm.value, fi.value, ms.value


def gen_stream(t, steps_mask, loops, out_of_place, pipelined):
    """Native task-stream generation -> (table int32[n,16], barriers int64[k])."""
    L = lib()
    n = ctypes.c_int64()
    nb = ctypes.c_int64()
    lp = loops.encode()
    check(L.tinv_gen_stream(t, steps_mask, lp, int(out_of_place), int(pipelined), None, 0, ctypes.byref(n),
                            None, 0, ctypes.byref(nb)))
    table = np.empty((n.value, TASK_FIELDS), dtype=np.int32)
    bars = np.empty(max(nb.value, 1), dtype=np.int64)
    check(L.tinv_gen_stream(t, steps_mask, lp, int(out_of_place), int(pipelined), _ip(table), n.value,
                            ctypes.byref(n), bars.ctypes.data_as(_I64P), len(bars), ctypes.byref(nb)))
    return table, bars[:nb.value].copy()


def dag_edges(table, barriers):
    """Native hazard scoreboard: (src, dst, kind) arrays, kind 0 RAW 1 WAR 2 WAW 3 barrier."""
    L = lib()
    table = np.ascontiguousarray(table, dtype=np.int32)
    bars = np.ascontiguousarray(barriers, dtype=np.int64)
    ne = ctypes.c_int64()
    check(L.tinv_dag_edges(_ip(table), len(table), _lp(bars), len(bars), None, None, None, 0, ctypes.byref(ne)))
    src = np.empty(ne.value, dtype=np.int32)
    dst = np.empty(ne.value, dtype=np.int32)
    kind = np.empty(ne.value, dtype=np.int8)
    check(L.tinv_dag_edges(_ip(table), len(table), _lp(bars), len(bars), _ip(src), _ip(dst),
                           kind.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), ne.value, ctypes.byref(ne)))
    return src, dst, kind


def dag_paths(table, barriers, weight=None, include_copies=False):
    """Native longest paths of the hazard DAG -> (best, via, depth, components);
    weight None: 1 per kernel task, 0 per COPY (include/tileinv_b200.h)."""
    L = lib()
    table = np.ascontiguousarray(table, dtype=np.int32)
    bars = np.ascontiguousarray(barriers, dtype=np.int64)
    n = len(table)
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float64)
    best = np.empty(n, dtype=np.float64)
    via = np.empty(n, dtype=np.int32)
    depth = np.empty(n, dtype=np.int32)
    nc = ctypes.c_int64()
    check(L.tinv_dag_paths(_ip(table), n, _lp(bars), len(bars), _dp(w) if w is not None else None,
                           int(include_copies), _dp(best), _ip(via), _ip(depth), ctypes.byref(nc)))
    return best, via, depth, nc.value


MODEL_COST_KEYS = ("blk", "item", "bpotrf", "btrtri", "bcopy", "send", "link", "mask", "hop")
# Item costs (us) of the schedule model, calibrated on the B200 (tools/scaling_model.py)
MODEL_COST = {"blk": 16.8, "item": 3.2, "bpotrf": 65.0, "btrtri": 10.7, "bcopy": 1.0, "send": 1.5, "link": 3.0,
              "mask": 0.6, "hop": 10.0}


KIND_NAMES = ("COPY", "POTRF", "TRSM", "SYRK_SUB", "SYRK_ADD_T", "GEMM", "TRTRI", "TRMM_LEFT", "TRMM_RIGHT_NEG",
              "TRMM_LEFT_T", "LAUUM", "INV", "SEND", "RECV", "ARRIVE", "DEPART", "POTRF_INV")


def model_run(n, b, table, t, barriers=(), aux=None, nrecv=0, rank_of=None, nranks=1, sms_per_rank=148,
              cost=None, with_crit=False, flags=0):
    """Schedule model (tinv_model_run, host only) -> (makespan us, busy SM-us per rank)."""
    L = lib()
    table = np.ascontiguousarray(table, dtype=np.int32)
    bars = np.ascontiguousarray(barriers, dtype=np.int64)
    cost = MODEL_COST if cost is None else cost
    c = np.array([cost[k] for k in MODEL_COST_KEYS], dtype=np.float64)
    out = np.zeros(nranks + 3, dtype=np.float64)
    ax = None if aux is None else np.ascontiguousarray(aux, dtype=np.int32)
    rk = None if rank_of is None else np.ascontiguousarray(rank_of, dtype=np.int32)
    crit = np.zeros(17, dtype=np.float64)
    check(L.tinv_model_run(n, b, _ip(table), len(table), t, _lp(bars), len(bars), _ip(ax), nrecv, _ip(rk), nranks,
                           sms_per_rank, flags, _dp(c), _dp(out), _dp(crit)))
    if out[nranks + 1] != 0:
        raise RuntimeError(f"model: {int(out[nranks + 1])} tasks never ran (deadlocked plan)")
    model_run.last_slots = int(out[nranks + 2])  # tile slots of the plan's device store
    if with_crit:
        return float(out[0]), out[1:nranks + 1].copy(), {KIND_NAMES[k]: float(crit[k]) for k in range(17) if crit[k]}
    return float(out[0]), out[1:nranks + 1].copy()


def dist_stream(table, t, P, Q):
    """Native distribution transform -> (table, owner, dest, ref) (include/tileinv_b200.h)."""
    L = lib()
    table = np.ascontiguousarray(table, dtype=np.int32)
    nout = ctypes.c_int64()
    check(L.tinv_dist_stream(_ip(table), len(table), t, P, Q, None, 0, ctypes.byref(nout), None, None, None))
    out = np.empty((nout.value, TASK_FIELDS), dtype=np.int32)
    owner = np.empty(nout.value, np.int32)
    dest = np.empty(nout.value, np.int32)
    ref = np.empty(nout.value, np.int32)
    check(L.tinv_dist_stream(_ip(table), len(table), t, P, Q, _ip(out), nout.value, ctypes.byref(nout), _ip(owner),
                             _ip(dest), _ip(ref)))
    return out, owner, dest, ref


class Context:
    """One device tile store (tinv_ctx) for an order-n matrix with tile order b."""

    def __init__(self, n, b, device=0, batch=1):
        L = lib()
        h = _P()
        rc = L.tinv_create_batch(ctypes.byref(h), batch, n, b, device)
        if rc != OK:
            raise NativeError(rc, last_error(None))
        self.h = h
        self.n, self.b, self.batch = n, b, batch
        self.t = n // b

    @classmethod
    def owned(cls, n, b, owned, device=0):
        """A partitioned store: slots only for the lower tiles with owned[i, j]
        != 0 (tinv_create_owned), e.g. one rank's 2D block-cyclic share."""
        self = cls.__new__(cls)
        own = np.ascontiguousarray(owned, dtype=np.int32)
        h = _P()
        rc = lib().tinv_create_owned(ctypes.byref(h), n, b, device, _ip(own))
        if rc != OK:
            raise NativeError(rc, last_error(None))
        self.h = h
        self.n, self.b, self.batch = n, b, 1
        self.t = n // b
        return self

    def recv_base(self):
        v = ctypes.c_int32()
        check(lib().tinv_recv_base(self.h, ctypes.byref(v)), self.h)
        return v.value

    def ipc_recv_bases(self, bases):
        arr = np.ascontiguousarray(bases, dtype=np.int32)
        check(lib().tinv_ipc_recv_bases(self.h, len(arr), _ip(arr)), self.h)

    def close(self):
        if self.h:
            lib().tinv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def store_bytes(self):
        v = ctypes.c_int64()
        check(lib().tinv_store_bytes(self.h, ctypes.byref(v)), self.h)
        return v.value

    def set_stream(self, stream_ptr):
        """Launch on a caller-owned cudaStream_t (int handle); 0 -> own stream."""
        check(lib().tinv_set_stream(self.h, ctypes.c_void_p(stream_ptr or None)), self.h)

    def ipc_open(self, rank, world, pool_handles, inbox_handles):
        check(lib().tinv_ipc_open(self.h, rank, world, b"".join(pool_handles), b"".join(inbox_handles)), self.h)

    def ipc_reset(self):
        check(lib().tinv_ipc_reset(self.h), self.h)

    def peer_attach(self, rank, contexts):
        """Map the peers' pools / inboxes by device pointer (ranks in one process, tinv_peer_attach)."""
        arr = (_P * len(contexts))(*[c.h for c in contexts])
        check(lib().tinv_peer_attach(self.h, rank, len(contexts), arr), self.h)

    def set_sms(self, nsm):
        """Executor grid of this context (tinv_set_sms)."""
        check(lib().tinv_set_sms(self.h, nsm), self.h)

    def put_dense(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64)
        check(lib().tinv_put_dense(self.h, _dp(m), m.shape[-1]), self.h)

    def get_dense(self, out, mode=DENSE_LOWER):
        assert out.dtype == np.float64 and out.flags["C_CONTIGUOUS"]
        check(lib().tinv_get_dense(self.h, _dp(out), out.shape[-1], mode), self.h)
        return out

    def put_dense_device(self, ptr, lda):
        check(lib().tinv_put_dense_device(self.h, ctypes.c_void_p(ptr), lda), self.h)

    def get_dense_device(self, ptr, lda, mode=DENSE_SYMMETRIZE):
        check(lib().tinv_get_dense_device(self.h, ctypes.c_void_p(ptr), lda, mode), self.h)

    def put_tile(self, i, j, tile):
        tile = np.ascontiguousarray(tile, dtype=np.float64)
        check(lib().tinv_put_tile(self.h, i, j, _dp(tile)), self.h)

    def get_tile(self, i, j):
        out = np.empty((self.b, self.b))
        check(lib().tinv_get_tile(self.h, i, j, _dp(out)), self.h)
        return out


class Plan:
    """A stream compiled for the device executor on one Context (reusable)."""

    def __init__(self, ctx, table, t, barriers, flags=0):
        L = lib()
        self.ctx = ctx
        self.table = np.ascontiguousarray(table, dtype=np.int32)
        self.barriers = np.ascontiguousarray(barriers, dtype=np.int64)
        self.h = _P()
        self.err = TinvErr()
        rc = L.tinv_plan_create(ctx.h, _ip(self.table), len(self.table), t, _lp(self.barriers),
                                len(self.barriers), flags, ctypes.byref(self.h), ctypes.byref(self.err))
        self.rc = rc
        self.msg = last_error(ctx.h) if rc != OK else ""

    @classmethod
    def xfer(cls, ctx, table, t, aux, nrecv, flags=0):
        """Plan with SEND / RECV transfer pseudo-tasks (tinv_plan_create_xfer)."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.table = np.ascontiguousarray(table, dtype=np.int32)
        self.barriers = np.zeros(0, np.int64)
        self.aux = np.ascontiguousarray(aux, dtype=np.int32)
        self.h = _P()
        self.err = TinvErr()
        self.rc = lib().tinv_plan_create_xfer(ctx.h, _ip(self.table), len(self.table), t, _ip(self.aux), nrecv, flags,
                                              ctypes.byref(self.h), ctypes.byref(self.err))
        self.msg = last_error(ctx.h) if self.rc != OK else ""
        return self

    @classmethod
    def ranks(cls, ctx, table, t, aux, nrecv, rank_of, nranks, flags=0):
        """Transfer plan with every rank's tasks run by its own CTA group in
        one launch (tinv_plan_create_ranks)."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.table = np.ascontiguousarray(table, dtype=np.int32)
        self.barriers = np.zeros(0, np.int64)
        self.aux = np.ascontiguousarray(aux, dtype=np.int32)
        self.rank_of = np.ascontiguousarray(rank_of, dtype=np.int32)
        self.h = _P()
        self.err = TinvErr()
        self.rc = lib().tinv_plan_create_ranks(ctx.h, _ip(self.table), len(self.table), t, _ip(self.aux), nrecv,
                                               _ip(self.rank_of), nranks, flags, ctypes.byref(self.h),
                                               ctypes.byref(self.err))
        self.msg = last_error(ctx.h) if self.rc != OK else ""
        return self

    def cta_idle(self):
        """-> (idle ns per CTA of the last run, rank of each CTA)."""
        g = ctypes.c_int64()
        check(lib().tinv_plan_cta_idle(self.h, None, None, 0, ctypes.byref(g)))
        idle = np.empty(g.value, np.int64)
        rank = np.empty(g.value, np.int32)
        check(lib().tinv_plan_cta_idle(self.h, idle.ctypes.data_as(_I64P), _ip(rank), g.value, ctypes.byref(g)))
        return idle, rank

    def run(self):
        """-> (rc, TinvErr, device ms)."""
        if self.rc != OK:
            return self.rc, self.err, 0.0
        ms = ctypes.c_double()
        rc = lib().tinv_plan_exec(self.h, ctypes.byref(self.err), ctypes.byref(ms))
        self.msg = last_error(self.ctx.h) if rc != OK else ""
        return rc, self.err, ms.value

    def run_host(self, a_ptr, lda, x_ptr, ldx, mode=DENSE_SYMMETRIZE):
        """Streamed end to end (STREAM_IO plans): host input -> executor -> host
        output, transfers overlapped with the computation. -> (rc, TinvErr, ms)."""
        if self.rc != OK:
            return self.rc, self.err, 0.0
        ms = ctypes.c_double()
        rc = lib().tinv_plan_exec_host(self.h, a_ptr, lda, x_ptr, ldx, mode, ctypes.byref(self.err),
                                       ctypes.byref(ms))
        self.msg = last_error(self.ctx.h) if rc != OK else ""
        return rc, self.err, ms.value

    def ipc_export(self):
        """-> (pool handle, inbox handle), 64 bytes each (CUDA IPC)."""
        hp = ctypes.create_string_buffer(64)
        hi = ctypes.create_string_buffer(64)
        check(lib().tinv_ipc_export(self.ctx.h, self.h, hp, hi), self.ctx.h)
        return hp.raw, hi.raw

    def stats(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().tinv_plan_stats(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"exec_tasks": a.value, "items": b.value, "edges": c.value}

    def trace(self):
        n = len(self.table)
        s = np.empty(n, np.int64)
        e = np.empty(n, np.int64)
        sm = np.empty(n, np.int32)
        check(lib().tinv_plan_trace(self.h, s.ctypes.data_as(_I64P), e.ctypes.data_as(_I64P), _ip(sm), n))
        return s, e, sm

    def close(self):
        if self.h:
            lib().tinv_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
