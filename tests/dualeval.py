"""Independent evaluation of an RLT2 dual state (test helper; shares nothing with the
oracle's C code or the CUDA library).

The dual objective of a permutation pi ("the cost of some
viable solution ... remains unchanged"):

  LB + sum_i b_{i pi(i)} + sum_{i != k} c_{i pi(i) k pi(k)}
     + sum_{ordered distinct (i,k,p)} d_{i pi(i), k pi(k), p pi(p)}

where the stored D block D{ij,kl} (i<k) stands for both logical blocks D_{ijkl} and
D_{klij}.  Layouts are the export layouts documented in
include/qap_rlt2.h.
"""
import itertools

import numpy as np


def block_index(n):
    idx = {}
    t = 0
    for i in range(n):
        for j in range(n):
            for k in range(i + 1, n):
                for l in range(n):
                    if l != j:
                        idx[(i, j, k, l)] = t
                        t += 1
    return idx


def skip1(x, a):
    return x - (x > a)


def skip2(x, a, b):
    return x - (x > a) - (x > b)


def d_logical(D, bidx, i, j, k, l, p, q):
    if i > k:
        i, j, k, l = k, l, i, j
    return D[bidx[(i, j, k, l)], skip2(p, i, k), skip2(q, j, l)]


def all_perms(n):
    return np.array(list(itertools.permutations(range(n))), dtype=np.int64)


def dual_values(n, lb, B, C, D, perms=None):
    """Dual objective for every permutation of the reduced problem (vectorised)."""
    if perms is None:
        perms = all_perms(n)
    B = np.asarray(B).reshape(n, n)
    C = np.asarray(C).reshape(n, n, n - 1, n - 1)
    D = np.asarray(D).reshape(-1, n - 2, n - 2)
    bidx = block_index(n)
    ar = np.arange(n)
    val = np.full(len(perms), float(lb))
    val += B[ar[None, :], perms].sum(axis=1)
    for i in range(n):
        for k in range(n):
            if i == k:
                continue
            val += C[i, perms[:, i], skip1(k, i), perms[:, k] - (perms[:, k] > perms[:, i])]
    # D: ordered distinct triples
    bl = np.full((n, n, n, n), -1, dtype=np.int64)
    for (i, j, k, l), t in bidx.items():
        bl[i, j, k, l] = t
    for i, k, p in itertools.permutations(range(n), 3):
        a, c = (i, k) if i < k else (k, i)
        ja, jc = (perms[:, a], perms[:, c])
        blk = bl[a, ja, c, jc]
        qp = perms[:, p]
        row = skip2(p, a, c)
        col = qp - (qp > ja).astype(np.int64) - (qp > jc).astype(np.int64)
        val += D[blk, row, col]
    return perms, val


def full_costs(F, Dist, perms):
    F = np.asarray(F)
    Dist = np.asarray(Dist)
    out = np.zeros(len(perms), dtype=np.int64)
    for i in range(F.shape[0]):
        for k in range(F.shape[0]):
            out += F[i, k] * Dist[perms[:, i], perms[:, k]]
    return out


def brute_force_opt(F, Dist):
    n = F.shape[0]
    best = None
    for chunk_first in range(n):
        rest = [x for x in range(n) if x != chunk_first]
        perms = np.array([(chunk_first,) + p for p in itertools.permutations(rest)], dtype=np.int64)
        c = full_costs(F, Dist, perms)
        m = int(c.min())
        best = m if best is None else min(best, m)
    return best


def gilmore_lawler(F, Dist, fixed=()):
    """Gilmore–Lawler bound from its textbook definition (sort-based minimal scalar
    products + an LAP), for the node with fixed pairs `fixed`."""
    from scipy.optimize import linear_sum_assignment
    F = np.asarray(F, dtype=np.int64)
    Dist = np.asarray(Dist, dtype=np.int64)
    N = F.shape[0]
    ff = {a for a, _ in fixed}
    fl = {b for _, b in fixed}
    I = [x for x in range(N) if x not in ff]
    J = [x for x in range(N) if x not in fl]
    kappa = sum(int(F[a, c]) * int(Dist[b, d]) for a, b in fixed for c, d in fixed)
    n = len(I)
    L = np.zeros((n, n), dtype=np.int64)
    for x, i in enumerate(I):
        for y, j in enumerate(J):
            lin = int(F[i, i]) * int(Dist[j, j])
            for a, b in fixed:
                lin += int(F[a, i]) * int(Dist[b, j]) + int(F[i, a]) * int(Dist[j, b])
            f = sorted(int(F[i, k]) for k in I if k != i)
            d = sorted((int(Dist[j, l]) for l in J if l != j), reverse=True)
            L[x, y] = lin + sum(a * b for a, b in zip(f, d))
    r, c = linear_sum_assignment(L)
    return kappa + int(L[r, c].sum())
