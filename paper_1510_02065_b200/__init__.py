"""Thin ctypes binding of libqaprlt2.so (include/qap_rlt2.h) — argument marshalling only.

Every step of the RLT2 bound runs in the library's CUDA kernels.  There is no CPU
fallback: if the shared library is missing or fails to load, importing the binding's
functions raises.  Function names are the C ABI's names.

    h = qap_rlt2_create(N, F, D)            # F, D: int64 N×N host arrays
    r = qap_rlt2_bound(h, max_iters=20)     # dict(lb, lb_glb, iters, status, ...)
    qap_rlt2_fix(h, [(fac, loc), ...])      # new node (cold)
    B, C, D, lb = qap_rlt2_dual_copy(h)     # export layouts of include/qap_rlt2.h
    qap_destroy(h)
"""
from __future__ import annotations

import ctypes as ct
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqaprlt2.so")

QAP_OK, QAP_E_ARG, QAP_E_CAPACITY, QAP_E_CUDA, QAP_E_NCCL, QAP_E_NUMERIC, QAP_E_STATE = range(7)
STATUS_NAMES = ["OK", "E_ARG", "E_CAPACITY", "E_CUDA", "E_NCCL", "E_NUMERIC", "E_STATE"]
QAP_FLAG_TIME_KERNELS = 1
QAP_FLAG_NO_GRAPH = 4
QAP_FLAG_LDG_TRANSFER = 8
PHASE_ITER0, PHASE_TRANSFER, PHASE_CONC_D, PHASE_CONC_C, PHASE_CONC_B = range(5)
KERNEL_KINDS = ["init", "sigma", "transfer", "lap2", "lap1", "lap0"]

EXPORTS = ["qap_rlt2_create", "qap_rlt2_load", "qap_rlt2_fix", "qap_rlt2_bound", "qap_rlt2_dual_sizes",
           "qap_rlt2_dual_copy", "qap_rlt2_step", "qap_rlt2_kernel_stats", "qap_last_error",
           "qap_destroy", "qap_lap_batch", "qap_bnb_solve", "qap_nccl_unique_id", "qap_rlt2_shard_info",
           "qap_shard_plan", "qap_rlt2_create_group", "qap_rlt2_group_bound", "qap_rlt2_bound_async",
           "qap_rlt2_bound_result", "qap_rlt2_strong_branch", "qap_bnb_run", "qap_bnb_frontier", "qap_rlt2_fold"]


class _BnbNode(ct.Structure):
    _fields_ = [("m", ct.c_int32), ("fac", ct.c_int32 * 64), ("loc", ct.c_int32 * 64), ("lb", ct.c_double)]


_SyncFn = ct.CFUNCTYPE(ct.c_int32, ct.c_void_p, ct.c_int64, ct.POINTER(ct.c_int32), ct.POINTER(ct.c_int64))
_DonateFn = ct.CFUNCTYPE(None, ct.c_void_p, ct.POINTER(_BnbNode))


class _BnbOpts(ct.Structure):
    _fields_ = [("iters", ct.c_int32), ("K", ct.c_double), ("UB0", ct.c_double), ("batch", ct.c_int32),
                ("sb_iters", ct.c_int32), ("checkpoint_path", ct.c_char_p), ("checkpoint_every", ct.c_int64),
                ("max_nodes", ct.c_int64), ("resume", ct.c_int32), ("root", ct.POINTER(_BnbNode)),
                ("sync", _SyncFn), ("donate", _DonateFn), ("ctx", ct.c_void_p), ("sync_every", ct.c_int64),
                ("warm", ct.c_int32)]


class _BnbResult(ct.Structure):
    _fields_ = [("opt", ct.c_int64), ("perm", ct.c_int32 * 64), ("bounded", ct.c_int64), ("leaves", ct.c_int64),
                ("pruned", ct.c_int64), ("sb_cut", ct.c_int64), ("complete", ct.c_int32),
                ("depth_max", ct.c_int32), ("open", ct.c_int64), ("bounded_by_depth", ct.c_int64 * 64)]


class QapError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


_XchgFn = ct.CFUNCTYPE(ct.c_int32, ct.c_void_p, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double),
                       ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64), ct.c_int32, ct.c_int32)
_GatherFn = ct.CFUNCTYPE(ct.c_int32, ct.c_void_p, ct.POINTER(ct.c_double), ct.POINTER(ct.c_int64), ct.c_int32,
                         ct.c_int32)


class _HostTransport(ct.Structure):
    _fields_ = [("ctx", ct.c_void_p), ("exchange", _XchgFn), ("allgather", _GatherFn)]


class _Opts(ct.Structure):
    _fields_ = [("device", ct.c_int32), ("cuda_stream", ct.c_void_p), ("flags", ct.c_int32),
                ("lap_warps", ct.c_int32), ("world", ct.c_int32), ("rank", ct.c_int32),
                ("nccl_id", ct.c_void_p), ("host_transport", ct.POINTER(_HostTransport))]


class _Result(ct.Structure):
    _fields_ = [("lb", ct.c_double), ("lb_glb", ct.c_double), ("iters", ct.c_int32),
                ("status", ct.c_int32), ("lb_trace", ct.POINTER(ct.c_double)),
                ("lb_trace_cap", ct.c_int32), ("launches", ct.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libqaprlt2.so (fails loudly if absent: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_1510_02065_b200.build` "
                          "(or __graft_entry__.build())")
    L = ct.CDLL(path)
    vp, i32, i64, f64 = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_double
    L.qap_rlt2_create.argtypes = [i32, vp, vp, ct.POINTER(_Opts), ct.POINTER(vp)]
    L.qap_rlt2_fix.argtypes = [vp, i32, vp, vp]
    L.qap_rlt2_load.argtypes = [vp, vp, vp]
    L.qap_rlt2_bound.argtypes = [vp, i32, f64, f64, ct.POINTER(_Result)]
    L.qap_rlt2_dual_sizes.argtypes = [vp, ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(i64)]
    L.qap_rlt2_dual_copy.argtypes = [vp, vp, vp, vp, ct.POINTER(f64)]
    L.qap_rlt2_step.argtypes = [vp, i32]
    L.qap_rlt2_kernel_stats.argtypes = [vp, vp, vp, i32]
    L.qap_last_error.argtypes = [vp]
    L.qap_last_error.restype = ct.c_char_p
    L.qap_destroy.argtypes = [vp]
    L.qap_destroy.restype = None
    L.qap_lap_batch.argtypes = [i32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.qap_bnb_solve.argtypes = [vp, i32, f64, f64, i32, i32, ct.POINTER(i64), vp, ct.POINTER(i64),
                                ct.POINTER(i64), ct.POINTER(i64), ct.POINTER(i64)]
    L.qap_rlt2_strong_branch.argtypes = [vp, i32, vp, ct.POINTER(i32), ct.POINTER(i32)]
    L.qap_bnb_run.argtypes = [vp, ct.POINTER(_BnbOpts), ct.POINTER(_BnbResult)]
    L.qap_rlt2_fold.argtypes = [vp, vp, i32, i32]
    L.qap_bnb_frontier.argtypes = [vp, ct.POINTER(_BnbOpts), i32, vp, i32, ct.POINTER(i32), ct.POINTER(_BnbResult)]
    L.qap_rlt2_bound_async.argtypes = [vp, i32, f64, f64]
    L.qap_rlt2_bound_result.argtypes = [vp, ct.POINTER(_Result)]
    L.qap_nccl_unique_id.argtypes = [vp]
    L.qap_rlt2_shard_info.argtypes = [vp] + [vp] * 7
    L.qap_shard_plan.argtypes = [i32, i32, i32, vp, vp, vp, vp, i64, ct.POINTER(i64)]
    L.qap_rlt2_create_group.argtypes = [i32, i32, vp, vp, ct.POINTER(_Opts), vp]
    L.qap_rlt2_group_bound.argtypes = [vp, i32, i32, f64, f64, vp]
    for name in EXPORTS:
        if name not in ("qap_last_error", "qap_destroy"):
            getattr(L, name).restype = ct.c_int
    _lib = L
    return L


def _check(st: int, h=None):
    if st != QAP_OK:
        msg = load_library().qap_last_error(h.ptr if isinstance(h, Handle) else h)
        raise QapError(st, (msg or b"").decode())


def _current_stream():
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:  # torch is plumbing only
        pass
    return None


class Handle:
    """Owner of a qap_rlt2* handle."""

    def __init__(self, ptr, N: int, world: int = 1):
        self.ptr = ptr
        self.N = N
        self.world = world  # > 1: a shard of a bound shared by `world` processes

    def close(self):
        if self.ptr:
            load_library().qap_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def host_transport(exchange, allgather):
    """qap_host_transport from two Python callables (argument marshalling only; the library
    stages its buffers to host memory around each call):
      exchange(send, recv, off, count, world, rank): numpy float64 views of the staged
        buffers and int64 arrays of per-peer offsets / counts (doubles);
      allgather(S_all, lo, world, rank): S_all in place, lo[world + 1].
    Keep the returned object alive as long as the handle (qap_rlt2_create does)."""
    def _x(_ctx, send, recv, off, cnt, world, rank):
        try:
            o = np.ctypeslib.as_array(off, (world,)).copy()
            c = np.ctypeslib.as_array(cnt, (world,)).copy()
            n = int((o + c).max()) if world else 0
            exchange(np.ctypeslib.as_array(send, (max(n, 1),)), np.ctypeslib.as_array(recv, (max(n, 1),)), o, c,
                     world, rank)
            return 0
        except BaseException:  # noqa: BLE001 - reported as a failed collective
            import traceback
            traceback.print_exc()
            return 1

    def _g(_ctx, S, lo, world, rank):
        try:
            lo_ = np.ctypeslib.as_array(lo, (world + 1,)).copy()
            allgather(np.ctypeslib.as_array(S, (max(int(lo_[-1]), 1),)), lo_, world, rank)
            return 0
        except BaseException:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1

    t = _HostTransport(None, _XchgFn(_x), _GatherFn(_g))
    t._keep = (t.exchange, t.allgather)
    return t


def qap_rlt2_create(N: int, F, D, device: int = -1, stream=None, flags: int = 0, lap_warps: int = 0,
                    world: int = 1, rank: int = 0, nccl_id: bytes | None = None, transport=None) -> Handle:
    """world > 1: this process's shard of one bound shared by `world` processes (collective;
    nccl_id = qap_nccl_unique_id() from rank 0, broadcast by the caller; or transport =
    host_transport(...) for host-staged collectives)."""
    L = load_library()
    F = np.ascontiguousarray(F, dtype=np.int64)
    D = np.ascontiguousarray(D, dtype=np.int64)
    if F.shape != (N, N) or D.shape != (N, N):
        raise ValueError("F and D must be N×N")
    idbuf = ct.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    opts = _Opts(device, stream if stream is not None else _current_stream(), flags, lap_warps, world, rank,
                 ct.cast(idbuf, ct.c_void_p) if idbuf is not None else None,
                 ct.pointer(transport) if transport is not None else None)
    out = ct.c_void_p()
    st = L.qap_rlt2_create(N, F.ctypes.data, D.ctypes.data, ct.byref(opts), ct.byref(out))
    _check(st, None)
    h = Handle(out.value, N, world)
    h._transport = transport  # the callbacks must outlive the handle
    return h


def qap_rlt2_load(h: Handle, F, D) -> None:
    """Replace the handle's instance (same N) from host arrays; resets to the root node."""
    F = np.ascontiguousarray(F, dtype=np.int64)
    D = np.ascontiguousarray(D, dtype=np.int64)
    if F.shape != (h.N, h.N) or D.shape != (h.N, h.N):
        raise ValueError("F and D must be N×N")
    _check(load_library().qap_rlt2_load(h.ptr, F.ctypes.data, D.ctypes.data), h)


def qap_rlt2_fix(h: Handle, fixed=()) -> None:
    fac = np.array([a for a, _ in fixed] or [0], dtype=np.int32)
    loc = np.array([b for _, b in fixed] or [0], dtype=np.int32)
    _check(load_library().qap_rlt2_fix(h.ptr, len(fixed), fac.ctypes.data, loc.ctypes.data), h)


def qap_rlt2_bound(h: Handle, max_iters: int, K: float = 0.0, UB: float = math.inf, trace: bool = False) -> dict:
    r = _Result()
    buf = None
    if trace and max_iters > 0:
        buf = (ct.c_double * max_iters)()
        r.lb_trace = ct.cast(buf, ct.POINTER(ct.c_double))
        r.lb_trace_cap = max_iters
    _check(load_library().qap_rlt2_bound(h.ptr, max_iters, K, UB, ct.byref(r)), h)
    out = dict(lb=r.lb, lb_glb=r.lb_glb, iters=r.iters, status=r.status, launches=r.launches)
    if buf is not None:
        out["trace"] = np.array(buf[: r.iters])
    return out


def qap_rlt2_dual_sizes(h: Handle):
    a, b, c = ct.c_int64(), ct.c_int64(), ct.c_int64()
    _check(load_library().qap_rlt2_dual_sizes(h.ptr, ct.byref(a), ct.byref(b), ct.byref(c)), h)
    return a.value, b.value, c.value


def qap_rlt2_dual_copy(h: Handle, want_B=True, want_C=True, want_D=True):
    nB, nC, nD = qap_rlt2_dual_sizes(h)
    B = np.empty(nB) if want_B else None
    C = np.empty(nC) if want_C else None
    D = np.empty(nD) if want_D else None
    lb = ct.c_double()
    _check(load_library().qap_rlt2_dual_copy(h.ptr, None if B is None else B.ctypes.data,
                                             None if C is None else C.ctypes.data,
                                             None if D is None else D.ctypes.data, ct.byref(lb)), h)
    return B, C, D, lb.value


def qap_rlt2_step(h: Handle, phase: int) -> None:
    _check(load_library().qap_rlt2_step(h.ptr, phase), h)


def qap_rlt2_kernel_stats(h: Handle, reset: bool = False) -> dict:
    n = len(KERNEL_KINDS)
    launches = np.zeros(n, np.int64)
    ms = np.zeros(n, np.float64)
    _check(load_library().qap_rlt2_kernel_stats(h.ptr, launches.ctypes.data, ms.ctypes.data, int(reset)), h)
    return {k: dict(launches=int(launches[i]), ms=float(ms[i])) for i, k in enumerate(KERNEL_KINDS)}


def qap_destroy(h: Handle) -> None:
    h.close()


def _ptr(t):
    return None if t is None else t.data_ptr()


def qap_lap_batch(M, R=None, S=None, assign=None, u=None, v=None, steps=None, err=None, stream=None):
    """Batched LAP on device tensors: M is (count, m, m) fp64 CUDA (torch) tensor; outputs
    are preallocated CUDA tensors or None.  Enqueued on `stream` (default: current)."""
    count, m, m2 = M.shape
    if m != m2 or M.stride(2) != 1 or M.stride(1) != m:
        raise ValueError("M must be (count, m, m) with row-major m×m matrices")
    ld = M.stride(0)
    st = load_library().qap_lap_batch(m, count, ld, _ptr(M), _ptr(R), _ptr(S), _ptr(assign), _ptr(u), _ptr(v),
                                      _ptr(steps), _ptr(err), stream if stream is not None else _current_stream())
    _check(st, None)


def qap_rlt2_bound_async(h: Handle, max_iters: int, K: float = 0.0, UB: float = math.inf) -> None:
    _check(load_library().qap_rlt2_bound_async(h.ptr, max_iters, K, UB), h)


def qap_rlt2_bound_result(h: Handle) -> dict:
    r = _Result()
    _check(load_library().qap_rlt2_bound_result(h.ptr, ct.byref(r)), h)
    return dict(lb=r.lb, lb_glb=r.lb_glb, iters=r.iters, status=r.status, launches=r.launches)


def qap_bnb_solve(h: Handle, iters: int, K: float = 0.0, UB0: float = math.inf, batch: int = 1,
                  sb_iters: int = -1, warm: bool = False) -> dict:
    if warm:  # warm children: through qap_bnb_run (the C signature of qap_bnb_solve is cold-only)
        r = qap_bnb_run(h, iters, K=K, UB0=UB0, batch=batch, sb_iters=sb_iters, warm=True)
        r.pop("complete")
        return r
    opt = ct.c_int64()
    perm = np.zeros(h.N, np.int32)
    b, l, p, c = ct.c_int64(), ct.c_int64(), ct.c_int64(), ct.c_int64()
    _check(load_library().qap_bnb_solve(h.ptr, iters, K, UB0, batch, sb_iters, ct.byref(opt), perm.ctypes.data,
                                        ct.byref(b), ct.byref(l), ct.byref(p), ct.byref(c)), h)
    return dict(opt=opt.value, perm=perm, bounded=b.value, leaves=l.value, pruned=p.value, sb_cut=c.value)


def qap_rlt2_fold(child: Handle, parent: Handle, fac: int, loc: int) -> None:
    """Warm child: child's node := parent's node + (fac at loc), state folded from the
    parent's current dual state (include/qap_rlt2.h, R31)."""
    _check(load_library().qap_rlt2_fold(child.ptr, parent.ptr, fac, loc), child)


def _node_in(nd: dict | None):
    """{"fac": [...], "loc": [...], "lb": float | nan} -> _BnbNode (or None)."""
    if nd is None:
        return None
    x = _BnbNode()
    x.m = len(nd["fac"])
    if x.m != len(nd["loc"]) or x.m > 64:
        raise ValueError("node: fac and loc of equal length <= 64")
    for t in range(x.m):
        x.fac[t], x.loc[t] = int(nd["fac"][t]), int(nd["loc"][t])
    x.lb = float(nd.get("lb", math.nan))
    return x


def _node_out(x) -> dict:
    return dict(fac=[x.fac[t] for t in range(x.m)], loc=[x.loc[t] for t in range(x.m)], lb=x.lb)


def _result_out(h: Handle, r) -> dict:
    return dict(opt=r.opt, perm=np.array(r.perm[: h.N], np.int32), bounded=r.bounded, leaves=r.leaves,
                pruned=r.pruned, sb_cut=r.sb_cut, complete=bool(r.complete), open=r.open, depth_max=r.depth_max,
                bounded_by_depth=[int(x) for x in r.bounded_by_depth[: h.N]])


def qap_bnb_run(h: Handle, iters: int, K: float = 0.0, UB0: float = math.inf, batch: int = 1,
                sb_iters: int = -1, checkpoint_path: str | None = None, checkpoint_every: int = 0,
                max_nodes: int = 0, resume: bool = False, root: dict | None = None, sync=None, donate=None,
                sync_every: int = 0, warm: bool = False) -> dict:
    """B&B with checkpoint/resume and the subtree-parallel hooks (include/qap_rlt2.h).
    root: {"fac", "loc", "lb"} — search only that subtree.  sync(local_best, perm | None) ->
    (global_best, n_donate); donate(node dict).  Exceptions raised in a callback abort the run
    and are re-raised here."""
    err = []

    def _sync(_ctx, best, perm, gout):
        try:
            g, k = sync(int(best), np.ctypeslib.as_array(perm, (h.N,)).copy() if perm else None)
            gout[0] = int(g)
            return int(k)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err.append(e)
            return -1

    def _donate(_ctx, nd):
        try:
            donate(_node_out(nd.contents))
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    rn = _node_in(root)
    cs = _SyncFn(_sync) if sync else _SyncFn()
    cd = _DonateFn(_donate) if donate else _DonateFn()
    o = _BnbOpts(iters, K, UB0, batch, sb_iters, checkpoint_path.encode() if checkpoint_path else None,
                 checkpoint_every, max_nodes, int(resume), ct.pointer(rn) if rn is not None else None, cs, cd, None,
                 sync_every, int(warm))
    r = _BnbResult()
    st = load_library().qap_bnb_run(h.ptr, ct.byref(o), ct.byref(r))
    if err:
        raise err[0]
    _check(st, h)
    return _result_out(h, r)


def qap_bnb_frontier(h: Handle, iters: int, target: int, K: float = 0.0, UB0: float = math.inf, batch: int = 1,
                     sb_iters: int = -1, root: dict | None = None, cap: int = 1 << 16):
    """Breadth-first expansion until a level holds >= target open nodes (include/qap_rlt2.h).
    Returns (open nodes in DFS order, result dict of the expansion)."""
    rn = _node_in(root)
    o = _BnbOpts(iters, K, UB0, batch, sb_iters, None, 0, 0, 0, ct.pointer(rn) if rn is not None else None,
                 _SyncFn(), _DonateFn(), None, 0, 0)
    nodes = (_BnbNode * cap)()
    n = ct.c_int32()
    r = _BnbResult()
    _check(load_library().qap_bnb_frontier(h.ptr, ct.byref(o), target, nodes, cap, ct.byref(n), ct.byref(r)), h)
    return [_node_out(nodes[k]) for k in range(n.value)], _result_out(h, r)


def qap_rlt2_strong_branch(h: Handle, sb_iters: int = 1):
    """RLT1 estimates of every candidate child of the current node (n×n) and the chosen line
    (kind 0 = row / 1 = column, reduced index)."""
    B, _, _ = qap_rlt2_dual_sizes(h)
    n = int(round(B ** 0.5))
    est = np.zeros(n * n, np.float64)
    kind, index = ct.c_int32(), ct.c_int32()
    _check(load_library().qap_rlt2_strong_branch(h.ptr, sb_iters, est.ctypes.data, ct.byref(kind),
                                                 ct.byref(index)), h)
    return est.reshape(n, n), kind.value, index.value


def qap_nccl_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    _check(load_library().qap_nccl_unique_id(buf), None)
    return buf.raw


def qap_rlt2_shard_info(h: Handle) -> dict:
    w, r = ct.c_int32(), ct.c_int32()
    lo, hi, tl, ts, sl = (ct.c_int64() for _ in range(5))
    _check(load_library().qap_rlt2_shard_info(h.ptr, ct.byref(w), ct.byref(r), ct.byref(lo), ct.byref(hi),
                                              ct.byref(tl), ct.byref(ts), ct.byref(sl)), h)
    return dict(world=w.value, rank=r.value, blk_lo=lo.value, blk_hi=hi.value, tiles_local=tl.value,
                tiles_shared=ts.value, slots=sl.value)


def qap_shard_plan(n: int, world: int, rank: int) -> dict:
    """Host-only shard plan (no GPU): block ranges, per-peer exchanged tiles, tile list."""
    L = load_library()
    cnt = ct.c_int64()
    blk = np.zeros(world + 1, np.int64)
    peer = np.zeros(world, np.int64)
    _check(L.qap_shard_plan(n, world, rank, blk.ctypes.data, peer.ctypes.data, None, None, 0, ct.byref(cnt)), None)
    tiles = np.zeros(max(cnt.value, 1), np.int32)
    tinfo = np.zeros(max(cnt.value, 1), np.int32)
    _check(L.qap_shard_plan(n, world, rank, None, None, tiles.ctypes.data, tinfo.ctypes.data, cnt.value,
                            ct.byref(cnt)), None)
    return dict(blk_lo=blk, peer_slots=peer, tiles=tiles[:cnt.value], kind=tinfo[:cnt.value] & 3,
                slot=tinfo[:cnt.value] >> 2)


class Group:
    """In-process group of G shards of one bound (single-GPU test vehicle of the sharded path)."""

    def __init__(self, G: int, N: int, F, D, device: int = -1, flags: int = 0, lap_warps: int = 0):
        L = load_library()
        F = np.ascontiguousarray(F, dtype=np.int64)
        D = np.ascontiguousarray(D, dtype=np.int64)
        opts = _Opts(device, _current_stream(), flags, lap_warps, G, 0, None)
        arr = (ct.c_void_p * G)()
        _check(L.qap_rlt2_create_group(G, N, F.ctypes.data, D.ctypes.data, ct.byref(opts), arr), None)
        self.G, self.N = G, N
        self.handles = [Handle(arr[r], N) for r in range(G)]
        self._arr = arr

    def fix(self, fixed=()):
        for h in self.handles:
            qap_rlt2_fix(h, fixed)

    def bound(self, max_iters: int, K: float = 0.0, UB: float = math.inf, trace: bool = False):
        G = self.G
        res = (_Result * G)()
        bufs = []
        for r in range(G):
            if trace and max_iters > 0:
                b = (ct.c_double * max_iters)()
                bufs.append(b)
                res[r].lb_trace = ct.cast(b, ct.POINTER(ct.c_double))
                res[r].lb_trace_cap = max_iters
        arr = (ct.c_void_p * G)(*[h.ptr for h in self.handles])
        _check(load_library().qap_rlt2_group_bound(arr, G, max_iters, K, UB, res), self.handles[0])
        out = []
        for r in range(G):
            d = dict(lb=res[r].lb, lb_glb=res[r].lb_glb, iters=res[r].iters, status=res[r].status)
            if bufs:
                d["trace"] = np.array(bufs[r][: res[r].iters])
            out.append(d)
        return out

    def dual(self):
        """B, C (replicated; from rank 0) and D assembled from every shard."""
        B, C, D, lb = qap_rlt2_dual_copy(self.handles[0])
        L = load_library()
        for h in self.handles[1:]:
            _check(L.qap_rlt2_dual_copy(h.ptr, None, None, D.ctypes.data, None), h)
        return B, C, D, lb

    def close(self):
        for h in self.handles:
            h.close()


class RLT2Bound:
    """Convenience owner: RLT2Bound(inst_F, inst_D).bound(20)."""

    def __init__(self, F, D, **kw):
        F = np.asarray(F)
        self.h = qap_rlt2_create(F.shape[0], F, D, **kw)

    def fix(self, fixed=()):
        qap_rlt2_fix(self.h, fixed)
        return self

    def bound(self, max_iters, K=0.0, UB=math.inf, trace=False):
        return qap_rlt2_bound(self.h, max_iters, K, UB, trace)

    def dual(self):
        return qap_rlt2_dual_copy(self.h)

    def close(self):
        self.h.close()
