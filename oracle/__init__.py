"""ctypes wrapper of the CPU oracle (``oracle/rlt2_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs — never by the product package
``paper_1510_02065_b200``.  It shares no code with the CUDA path.

Parity status per function (DESIGN.md §4 lists the pins):
  lap                   pinned: brute force (m<=8), scipy LAP value, LP certificate,
                        Bellman–Ford canonical dual (tests/test_oracle_lap.py)
  iteration0 (GLB)      pinned: closed-form Gilmore–Lawler bound (tests/test_oracle_rlt2.py)
  spread / transfer /   pinned: preservation over all permutations (n<=6), class-sum
  concentrate steps     conservation, idempotence, nonnegativity, worked examples
  bound                 pinned: LB <= brute-force OPT (N<=9), monotone, constant-cost
                        instances reach OPT exactly; terminal values at N>=10 are
                        "parity unpinned" beyond these validity properties
  bnb                   pinned: optimum == brute-force optimum (N<=9)
  fold (warm child)     pinned: preservation of every completion's cost and nonnegativity
                        (exhaustive, n<=6), LB(child) >= LB(parent), warm B&B optimum ==
                        brute force (tests/test_oracle_warm.py)
"""
from __future__ import annotations

import ctypes as ct
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rlt2_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off, no intrinsics; OpenMP for the
    optional all-cores mode, 1 thread unless set_threads() raises it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ct.CDLL(build())
        L.oracle_lap.argtypes = [ct.c_int, _f64p, _f64p, _i32p, _f64p, _f64p,
                                 ct.POINTER(ct.c_double), ct.POINTER(ct.c_int64)]
        L.oracle_lap_bruteforce.argtypes = [ct.c_int, _f64p, ct.POINTER(ct.c_double), _i32p]
        L.oracle_state_new.restype = ct.c_void_p
        L.oracle_state_new.argtypes = [ct.c_int, _i64p, _i64p, ct.c_int, _i32p, _i32p,
                                       ct.POINTER(ct.c_int)]
        L.oracle_state_free.argtypes = [ct.c_void_p]
        for f in ("oracle_iteration0", "oracle_spread_b", "oracle_spread_c_transfer_d",
                  "oracle_concentrate_d", "oracle_transfer_c", "oracle_concentrate_c"):
            getattr(L, f).argtypes = [ct.c_void_p]
        L.oracle_concentrate_b.argtypes = [ct.c_void_p, ct.POINTER(ct.c_double)]
        L.oracle_iteration.argtypes = [ct.c_void_p, ct.POINTER(ct.c_double)]
        L.oracle_bound.argtypes = [ct.c_void_p, ct.c_int, ct.c_double, ct.c_double,
                                   ct.POINTER(ct.c_double), ct.POINTER(ct.c_double),
                                   ct.POINTER(ct.c_int), ct.POINTER(ct.c_int), ct.c_void_p]
        L.oracle_state_n.argtypes = [ct.c_void_p]
        L.oracle_state_kappa.argtypes = [ct.c_void_p]
        L.oracle_state_kappa.restype = ct.c_int64
        L.oracle_state_lb_dual.argtypes = [ct.c_void_p]
        L.oracle_state_lb_dual.restype = ct.c_double
        L.oracle_state_lb_glb.argtypes = [ct.c_void_p]
        L.oracle_state_lb_glb.restype = ct.c_double
        L.oracle_state_sizes.argtypes = [ct.c_void_p] + [ct.POINTER(ct.c_int64)] * 3
        for f in ("oracle_state_B", "oracle_state_C", "oracle_state_D"):
            getattr(L, f).argtypes = [ct.c_void_p]
            getattr(L, f).restype = ct.POINTER(ct.c_double)
        L.oracle_state_free_maps.argtypes = [ct.c_void_p, _i32p, _i32p]
        L.oracle_state_fold.restype = ct.c_void_p
        L.oracle_state_fold.argtypes = [ct.c_void_p, ct.c_int, ct.c_int, ct.POINTER(ct.c_int)]
        L.oracle_bnb.argtypes = [ct.c_int, _i64p, _i64p, ct.c_int, ct.c_double, ct.c_double, ct.c_int, ct.c_int,
                                 ct.POINTER(ct.c_int64), _i32p, ct.POINTER(ct.c_int64),
                                 ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64)]
        L.oracle_rlt1_iteration.argtypes = [ct.c_void_p, ct.POINTER(ct.c_double)]
        L.oracle_rlt1_bound.argtypes = [ct.c_void_p, ct.c_int, ct.POINTER(ct.c_double)]
        L.oracle_strong_branch.argtypes = [ct.c_int, _i64p, _i64p, ct.c_int, _i32p, _i32p, ct.c_int, _f64p,
                                           ct.POINTER(ct.c_int), ct.POINTER(ct.c_int)]
        L.oracle_set_threads.argtypes = [ct.c_int]
        L.oracle_qap_bruteforce.argtypes = [ct.c_int, _i64p, _i64p, ct.POINTER(ct.c_int64), _i32p]
        _lib = L
    return _lib


def set_threads(t: int) -> None:
    """Host threads for the independent units of each step (1 = the plain sequential oracle;
    every thread count gives bit-identical results)."""
    lib().oracle_set_threads(int(t))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st:
        raise OracleError(f"{what} failed with status {st}")


def lap(M):
    """O2: returns dict(S, assign, u, v, R, steps) for the m×m fp64 matrix M."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    m = M.shape[0]
    R = np.empty_like(M)
    a = np.empty(m, np.int32)
    u = np.empty(m, np.float64)
    v = np.empty(m, np.float64)
    S = ct.c_double()
    steps = ct.c_int64()
    _check(lib().oracle_lap(m, M, R, a, u, v, ct.byref(S), ct.byref(steps)), "oracle_lap")
    return dict(S=S.value, assign=a, u=u, v=v, R=R, steps=steps.value)


def lap_bruteforce(M):
    M = np.ascontiguousarray(M, dtype=np.float64)
    m = M.shape[0]
    best = ct.c_double()
    a = np.empty(m, np.int32)
    _check(lib().oracle_lap_bruteforce(m, M, ct.byref(best), a), "oracle_lap_bruteforce")
    return best.value, a


class State:
    """The dual state (B, C, D, LB) of one node; O0/O1 at construction."""

    def __init__(self, F, Dist, fixed=()):
        F = np.ascontiguousarray(F, dtype=np.int64)
        Dist = np.ascontiguousarray(Dist, dtype=np.int64)
        N = F.shape[0]
        fac = np.array([p[0] for p in fixed] or [0], dtype=np.int32)
        loc = np.array([p[1] for p in fixed] or [0], dtype=np.int32)
        err = ct.c_int()
        self._L = lib()
        self._h = self._L.oracle_state_new(N, F, Dist, len(fixed), fac, loc, ct.byref(err))
        if not self._h:
            raise OracleError(f"oracle_state_new failed with status {err.value}")
        self.N = N
        self.n = self._L.oracle_state_n(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.oracle_state_free(h)
            self._h = None

    # steps ---------------------------------------------------------------
    def iteration0(self):
        _check(self._L.oracle_iteration0(self._h), "iteration0")

    def spread_b(self):
        _check(self._L.oracle_spread_b(self._h), "spread_b")

    def spread_c_transfer_d(self):
        _check(self._L.oracle_spread_c_transfer_d(self._h), "spread_c_transfer_d")

    def concentrate_d(self):
        _check(self._L.oracle_concentrate_d(self._h), "concentrate_d")

    def transfer_c(self):
        _check(self._L.oracle_transfer_c(self._h), "transfer_c")

    def concentrate_c(self):
        _check(self._L.oracle_concentrate_c(self._h), "concentrate_c")

    def concentrate_b(self) -> float:
        x = ct.c_double()
        _check(self._L.oracle_concentrate_b(self._h, ct.byref(x)), "concentrate_b")
        return x.value

    def rlt1_iteration(self) -> float:
        x = ct.c_double()
        _check(self._L.oracle_rlt1_iteration(self._h, ct.byref(x)), "rlt1_iteration")
        return x.value

    def rlt1_bound(self, T: int) -> float:
        x = ct.c_double()
        _check(self._L.oracle_rlt1_bound(self._h, T, ct.byref(x)), "rlt1_bound")
        return x.value

    def iteration(self) -> float:
        x = ct.c_double()
        _check(self._L.oracle_iteration(self._h, ct.byref(x)), "iteration")
        return x.value

    def bound(self, T: int, K: float = 0.0, UB: float = math.inf, trace: bool = False):
        lb, glb = ct.c_double(), ct.c_double()
        it, st = ct.c_int(), ct.c_int()
        tr = np.zeros(max(T, 1), np.float64)
        _check(self._L.oracle_bound(self._h, T, K, UB, ct.byref(lb), ct.byref(glb), ct.byref(it),
                                    ct.byref(st), tr.ctypes.data_as(ct.c_void_p)), "bound")
        out = dict(lb=lb.value, lb_glb=glb.value, iters=it.value, status=st.value)
        if trace:
            out["trace"] = tr[: it.value].copy()
        return out

    # state ---------------------------------------------------------------
    @property
    def kappa(self) -> int:
        return int(self._L.oracle_state_kappa(self._h))

    @property
    def lb_dual(self) -> float:
        return self._L.oracle_state_lb_dual(self._h)

    @property
    def lb(self) -> float:
        return float(self.kappa) + self.lb_dual

    def _arr(self, f, count):
        p = f(self._h)
        return np.ctypeslib.as_array(p, shape=(count,))

    def sizes(self):
        a, b, c = ct.c_int64(), ct.c_int64(), ct.c_int64()
        self._L.oracle_state_sizes(self._h, ct.byref(a), ct.byref(b), ct.byref(c))
        return a.value, b.value, c.value

    @property
    def B(self) -> np.ndarray:
        """Live view (n×n)."""
        n = self.n
        return self._arr(self._L.oracle_state_B, n * n).reshape(n, n)

    @property
    def C(self) -> np.ndarray:
        """Live view (n, n, n-1, n-1): C[i, j] is block C_ij."""
        n = self.n
        return self._arr(self._L.oracle_state_C, self.sizes()[1]).reshape(n, n, n - 1, n - 1)

    @property
    def D(self) -> np.ndarray:
        """Live view (nblk, n-2, n-2) in canonical (i,j,k,l), i<k, l!=j block order."""
        n = self.n
        nD = self.sizes()[2]
        return self._arr(self._L.oracle_state_D, nD).reshape(-1, n - 2, n - 2)

    def fold(self, a: int, b: int) -> "State":
        """Warm child fixing reduced facility a at reduced location b (NEXT-3, reading R31)."""
        err = ct.c_int()
        h = self._L.oracle_state_fold(self._h, a, b, ct.byref(err))
        if not h:
            raise OracleError(f"oracle_state_fold failed with status {err.value}")
        c = State.__new__(State)
        c._L, c._h, c.N, c.n = self._L, h, self.N, self._L.oracle_state_n(h)
        return c

    def free_maps(self):
        I = np.empty(self.n, np.int32)
        J = np.empty(self.n, np.int32)
        self._L.oracle_state_free_maps(self._h, I, J)
        return I, J


def bound(F, Dist, T: int, K: float = 0.0, UB: float = math.inf, fixed=(), trace=False):
    s = State(F, Dist, fixed)
    return s.bound(T, K, UB, trace=trace)


def bnb(F, Dist, T: int = 3, K: float = 0.0, UB0: float = math.inf, sb_iters: int = -1, warm: bool = False):
    """Minimal deterministic DFS branch-and-bound (strong branching with RLT1 when
    sb_iters >= 0; warm children folded from the parent's state when warm); returns
    dict(opt, perm, bounded, leaves, pruned, sb_cut)."""
    F = np.ascontiguousarray(F, dtype=np.int64)
    Dist = np.ascontiguousarray(Dist, dtype=np.int64)
    N = F.shape[0]
    best = ct.c_int64()
    perm = np.zeros(N, np.int32)
    b, l, p, c = ct.c_int64(), ct.c_int64(), ct.c_int64(), ct.c_int64()
    _check(lib().oracle_bnb(N, F, Dist, T, K, UB0, sb_iters, int(warm), ct.byref(best), perm, ct.byref(b), ct.byref(l),
                            ct.byref(p), ct.byref(c)), "bnb")
    return dict(opt=best.value, perm=perm, bounded=b.value, leaves=l.value, pruned=p.value, sb_cut=c.value)


def qap_bruteforce(F, Dist):
    """Brute-force QAP optimum over all N! permutations (test pin; N <= 13): (opt, first
    permutation in lexicographic order reaching it)."""
    F = np.ascontiguousarray(F, dtype=np.int64)
    Dist = np.ascontiguousarray(Dist, dtype=np.int64)
    N = F.shape[0]
    best = ct.c_int64()
    perm = np.zeros(N, np.int32)
    _check(lib().oracle_qap_bruteforce(N, F, Dist, ct.byref(best), perm), "qap_bruteforce")
    return best.value, perm


def strong_branch(F, Dist, fixed=(), T: int = 1):
    """RLT1 estimates est[a, b] of every candidate child and the selected line (kind 0 = row /
    1 = column, reduced index)."""
    F = np.ascontiguousarray(F, dtype=np.int64)
    Dist = np.ascontiguousarray(Dist, dtype=np.int64)
    N = F.shape[0]
    n = N - len(fixed)
    fac = np.array([a for a, _ in fixed] or [0], dtype=np.int32)
    loc = np.array([b for _, b in fixed] or [0], dtype=np.int32)
    est = np.zeros(n * n, np.float64)
    kind, index = ct.c_int(), ct.c_int()
    _check(lib().oracle_strong_branch(N, F, Dist, len(fixed), fac, loc, T, est, ct.byref(kind), ct.byref(index)),
           "strong_branch")
    return est.reshape(n, n), kind.value, index.value


def block_list(n: int):
    """Canonical stored-block enumeration (i,j,k,l), i<k, l!=j — the export layout order."""
    return [(i, j, k, l) for i in range(n) for j in range(n) for k in range(i + 1, n)
            for l in range(n) if l != j]
