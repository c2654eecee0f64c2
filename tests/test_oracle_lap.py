"""Pins of the oracle's LAP (O2) against things other than itself:
brute-force enumeration, scipy's LAP, the LP optimality certificate, the canonical-dual
characterisation (reading R5, recomputed by Bellman–Ford) and SPEC worked
examples (tests/golden/spec_examples.json)."""
import itertools
import json
import os

import numpy as np
import pytest
from scipy.optimize import linear_sum_assignment

import qapgen

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def certificate_ok(M, out, exact):
    m = M.shape[0]
    a, u, v, R = out["assign"], out["u"], out["v"], out["R"]
    assert sorted(a.tolist()) == list(range(m)), "assignment is a bijection"
    scale = max(1.0, np.abs(M).max())
    assert (R >= 0).all()
    assert all(R[r, a[r]] == 0 for r in range(m))
    raw = (M - u[:, None]) - v[None, :]
    tol = 0 if exact else 1e-12 * scale
    assert np.abs(np.where(R == 0, 0, raw - R)).max() <= tol
    assert raw.min() >= -1e-9 * scale
    primal = sum(M[r, a[r]] for r in range(m))
    assert abs(out["S"] - primal) <= (0 if exact else 1e-12 * scale * m)
    assert abs(u.sum() + v.sum() - out["S"]) <= (0 if exact else 1e-11 * scale * m)


def canonical_v(M, assign):
    """Largest v <= 0 with v_s - v_{pi(r)} <= M[r][s] - M[r][pi(r)] (Bellman–Ford)."""
    m = M.shape[0]
    v = np.zeros(m)
    for _ in range(m + 1):
        changed = False
        for r in range(m):
            pr = assign[r]
            for s in range(m):
                cand = v[pr] + (M[r, s] - M[r, pr])
                if cand < v[s]:
                    v[s] = cand
                    changed = True
        if not changed:
            break
    return v


@pytest.mark.parametrize("case", GOLDEN["lap"], ids=lambda c: c["cite"][:12])
def test_golden_examples(orc, case):
    M = np.array(case["M"], dtype=np.float64)
    out = orc.lap(M)
    assert out["S"] == case["S"]
    certificate_ok(M, out, exact=True)


@pytest.mark.parametrize("kind", ["int", "rank1", "zeros", "real"])
@pytest.mark.parametrize("m", [1, 2, 3, 5, 6, 8])
def test_bruteforce(orc, kind, m):
    for seed in range(6 if m == 8 else 15):
        M = qapgen.random_matrix(m, seed, kind)
        out = orc.lap(M)
        best, _ = orc.lap_bruteforce(M)
        # independent enumeration in Python as well
        if m <= 6:
            py = min(sum(M[r, p[r]] for r in range(m)) for p in itertools.permutations(range(m)))
            assert abs(py - best) <= 1e-12 * max(1, abs(best))
        exact = kind != "real"
        if exact:
            assert out["S"] == best
        else:
            assert abs(out["S"] - best) <= 1e-12 * max(1.0, best)
        assert abs(sum(M[r, out["assign"][r]] for r in range(m)) - best) <= (0 if exact else 1e-12 * max(1.0, best))
        certificate_ok(M, out, exact)


@pytest.mark.parametrize("kind", ["int", "rank1", "zeros", "real"])
@pytest.mark.parametrize("m", [10, 18, 28, 38])
def test_scipy_value(orc, kind, m):
    for seed in range(4):
        M = qapgen.random_matrix(m, seed, kind, hi=1000)
        out = orc.lap(M)
        r, c = linear_sum_assignment(M)
        ref = M[r, c].sum()
        if kind == "real":
            assert abs(out["S"] - ref) <= 1e-12 * max(1.0, ref) * m
        else:
            assert out["S"] == ref
        certificate_ok(M, out, exact=(kind != "real"))


@pytest.mark.parametrize("kind", ["int", "rank1", "zeros", "real"])
@pytest.mark.parametrize("m", [3, 5, 8, 12, 20])
def test_canonical_dual(orc, kind, m):
    """Reading R5: the cold-start SAP dual is the v-maximal dual with v <= 0."""
    for seed in range(5):
        M = qapgen.random_matrix(m, seed + 100, kind)
        out = orc.lap(M)
        vstar = canonical_v(M, out["assign"])
        assert (vstar <= 0).all()
        tol = 0 if kind != "real" else 1e-12 * max(1.0, np.abs(M).max())
        assert np.abs(out["v"] - vstar).max() <= tol


def test_residual_fixpoint(orc):
    """LAP on the residual returns value 0."""
    for seed in range(5):
        M = qapgen.random_matrix(12, seed, "real")
        R = orc.lap(M)["R"]
        assert orc.lap(R)["S"] == 0.0


def test_tie_rule_prefers_free_column(orc):
    """Reading R6: on an all-zero matrix row 0 takes column 0 in the row reduction (every
    row's lowest minimum column is 0) and every later row takes a free column at once: one
    Dijkstra step per remaining row and the identity assignment."""
    out = orc.lap(np.zeros((7, 7)))
    assert out["steps"] == 6
    assert out["assign"].tolist() == list(range(7))


def test_nonnegative_and_zero_canonical(orc):
    M = qapgen.random_matrix(9, 3, "zeros")
    R = orc.lap(M)["R"]
    assert not np.signbit(R).any(), "no -0.0 in residuals"
