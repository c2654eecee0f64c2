"""Seeded synthetic QAP instance generators (shared by the oracle tests and the GPU path).

This module holds NO arithmetic of the RLT2 method: it only draws integer flow and
distance matrices.  Both sides of every parity test read the same int64 matrices
produced here (or the same QAPLIB ``.dat`` bytes written by :func:`write_dat`).

Families:

* ``nug``  — Nugent-shaped (Table 1 nug* rows): Manhattan distances
  on an r×c grid, symmetric zero-diagonal flows, each unordered facility pair has flow 0
  with probability 1/2, else U{1..10}.
* ``taib`` — tai*b-shaped (Table 1 tai*b rows): grid Manhattan
  distances ×10, asymmetric zero-diagonal clustered flows.  A seeded shuffle puts
  facilities into clusters of 5; intra-cluster flows are nonzero w.p. 0.8 with value
  U{10..999}, inter-cluster flows nonzero w.p. 0.1 with value U{1..99}.
* ``uniform`` — dense U{0..hi} flows and distances with zero diagonals (test family).
* ``const``  — constant-cost instance: f_ik = 1 for i≠k, random distances; every
  permutation has the same cost (closed-form pin).
* ``zero``   — all-zero instance.

RNG: splitmix64(seed); ``U{a..b} = a + next() mod (b-a+1)``.  Everything is integer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_MASK = (1 << 64) - 1


class SplitMix64:
    """Counter-based splitmix64 stream (Steele, Lea & Flood 2014)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def uniform(self, a: int, b: int) -> int:
        """U{a..b} inclusive."""
        return a + self.next() % (b - a + 1)


GRID_SHAPES = {8: (2, 4), 12: (3, 4), 20: (4, 5), 30: (5, 6), 35: (5, 7), 40: (5, 8)}


def grid_shape(n: int) -> tuple[int, int]:
    """Rows × cols of the location grid: the table above, else the most square factorisation."""
    if n in GRID_SHAPES:
        return GRID_SHAPES[n]
    r = int(math.isqrt(n))
    while r > 1 and n % r:
        r -= 1
    return r, n // r


def manhattan(n: int, scale: int = 1) -> np.ndarray:
    r, c = grid_shape(n)
    pos = [(j // c, j % c) for j in range(n)]
    d = np.zeros((n, n), dtype=np.int64)
    for a in range(n):
        for b in range(n):
            d[a, b] = scale * (abs(pos[a][0] - pos[b][0]) + abs(pos[a][1] - pos[b][1]))
    return d


@dataclass
class Instance:
    name: str
    n: int
    F: np.ndarray   # int64 n×n flows f_ik
    D: np.ndarray   # int64 n×n distances d_jl

    def evaluate(self, perm) -> int:
        """QAPLIB objective sum_{i,k} f_ik d_{p(i)p(k)} (diagonal included)."""
        p = np.asarray(perm, dtype=np.int64)
        return int((self.F * self.D[np.ix_(p, p)]).sum())


def nug(n: int, seed: int = 1) -> Instance:
    rng = SplitMix64(seed)
    F = np.zeros((n, n), dtype=np.int64)
    for i in range(n):
        for k in range(i + 1, n):
            if rng.next() % 2 == 0:
                v = 0
            else:
                v = rng.uniform(1, 10)
            F[i, k] = F[k, i] = v
    return Instance(f"nug{n}s{seed}", n, F, manhattan(n))


def taib(n: int, seed: int = 1) -> Instance:
    rng = SplitMix64(seed)
    order = list(range(n))
    for a in range(n - 1, 0, -1):          # Fisher–Yates
        b = rng.next() % (a + 1)
        order[a], order[b] = order[b], order[a]
    cluster = [0] * n
    for pos, fac in enumerate(order):
        cluster[fac] = pos // 5
    F = np.zeros((n, n), dtype=np.int64)
    for i in range(n):
        for k in range(n):
            if i == k:
                continue
            if cluster[i] == cluster[k]:
                F[i, k] = rng.uniform(10, 999) if rng.next() % 5 != 0 else 0
            else:
                F[i, k] = rng.uniform(1, 99) if rng.next() % 10 == 0 else 0
    return Instance(f"taib{n}s{seed}", n, F, manhattan(n, 10))


def uniform(n: int, seed: int = 1, hi: int = 20) -> Instance:
    rng = SplitMix64(seed)
    F = np.zeros((n, n), dtype=np.int64)
    D = np.zeros((n, n), dtype=np.int64)
    for i in range(n):
        for k in range(n):
            if i != k:
                F[i, k] = rng.uniform(0, hi)
    for i in range(n):
        for k in range(n):
            if i != k:
                D[i, k] = rng.uniform(0, hi)
    return Instance(f"unif{n}s{seed}", n, F, D)


def const(n: int, seed: int = 1) -> Instance:
    F = np.ones((n, n), dtype=np.int64) - np.eye(n, dtype=np.int64)
    return Instance(f"const{n}s{seed}", n, F, uniform(n, seed).D)


def zero(n: int) -> Instance:
    z = np.zeros((n, n), dtype=np.int64)
    return Instance(f"zero{n}", n, z, z.copy())


FAMILIES = {"nug": nug, "taib": taib, "uniform": uniform, "const": const}


def make(family: str, n: int, seed: int = 1) -> Instance:
    if family == "zero":
        return zero(n)
    return FAMILIES[family](n, seed)


def random_matrix(m: int, seed: int, kind: str = "int", hi: int = 100) -> np.ndarray:
    """Seeded m×m LAP test matrices (fp64): 'int' U{0..hi}, 'real' U[0,hi) with 52-bit
    mantissas, 'rank1' f⊗d integer outer product, 'zeros' 70% exact zeros."""
    rng = SplitMix64(seed * 1000003 + m)
    M = np.zeros((m, m), dtype=np.float64)
    if kind == "int":
        for r in range(m):
            for s in range(m):
                M[r, s] = rng.uniform(0, hi)
    elif kind == "real":
        for r in range(m):
            for s in range(m):
                M[r, s] = (rng.next() >> 11) * (hi / float(1 << 53))
    elif kind == "rank1":
        f = [rng.uniform(0, hi) for _ in range(m)]
        d = [rng.uniform(0, hi) for _ in range(m)]
        for r in range(m):
            for s in range(m):
                M[r, s] = float(f[r] * d[s])
    elif kind == "zeros":
        for r in range(m):
            for s in range(m):
                M[r, s] = 0.0 if rng.next() % 10 < 7 else float(rng.uniform(1, hi))
    else:
        raise ValueError(kind)
    return M


def write_dat(inst: Instance, path) -> None:
    """QAPLIB .dat: n, then F row-major, then D row-major."""
    with open(path, "w") as fh:
        fh.write(f"{inst.n}\n\n")
        for mat in (inst.F, inst.D):
            for row in mat:
                fh.write(" ".join(str(int(x)) for x in row) + "\n")
            fh.write("\n")


def read_dat(path, name: str | None = None) -> Instance:
    toks = open(path).read().split()
    n = int(toks[0])
    if len(toks) != 1 + 2 * n * n:
        raise ValueError(f"expected {1 + 2 * n * n} integers, found {len(toks)}")
    vals = np.array([int(t) for t in toks[1:]], dtype=np.int64)
    if (vals < 0).any():
        raise ValueError("negative entry")
    return Instance(name or str(path), n, vals[: n * n].reshape(n, n), vals[n * n:].reshape(n, n))
