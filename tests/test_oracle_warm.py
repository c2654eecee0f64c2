"""Pins of the oracle's warm child (oracle_state_fold, DESIGN.md
reading R31) and the warm B&B, against what the mathematics fixes:

* preservation: for every completion of the child, the child state's dual objective
  equals the full permutation's cost — exhaustively, for every child (a, b) of parents at
  n = 4..6 bounded for 0..2 iterations, and again after every step of the child's own ascent;
* nonnegativity of every entry;
* LB(child) >= LB(parent) (b_ab >= 0 and every concentration adds S >= 0) and
  LB(child) <= the best completion of the child (validity, brute force);
* constant-cost instances: a warm child's bound equals the (common) optimum;
* the warm B&B optimum equals brute force (N <= 9), with and without strong branching.
A dropped or mis-indexed fold term, a wrong multiplicity of the D terms or a transposed
C operand breaks preservation.
"""
import itertools

import numpy as np
import pytest

import qapgen
from tests import dualeval as de
from tests.test_oracle_rlt2 import STEPS, check_nonneg, check_preservation


def child_fixed(st, fixed, a, b):
    I, J = st.free_maps()
    return list(fixed) + [(int(I[a]), int(J[b]))]


def subtree_opt(inst, fixed):
    N = inst.n
    ff = [f for f, _ in fixed]
    fl = [l for _, l in fixed]
    I = [x for x in range(N) if x not in ff]
    J = [x for x in range(N) if x not in fl]
    best = None
    for p in itertools.permutations(J):
        perm = [0] * N
        for f, l in fixed:
            perm[f] = l
        for x, y in zip(I, p):
            perm[x] = y
        v = inst.evaluate(perm)
        best = v if best is None else min(best, v)
    return best


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
@pytest.mark.parametrize("n,T", [(4, 0), (5, 1), (6, 2), (6, 0)])
def test_fold_preserves_every_completion(orc, family, n, T):
    for seed in (1, 2):
        inst = qapgen.make(family, n, seed)
        par = orc.State(inst.F, inst.D)
        rp = par.bound(T)
        for a in range(n):
            for b in range(n):
                ch = par.fold(a, b)
                fx = child_fixed(par, (), a, b)
                assert ch.n == n - 1 and ch.kappa == par.kappa
                assert ch.lb == par.lb + float(par.B[a, b])          # lb' = lb + b_ab
                check_preservation(ch, inst, fixed=fx)
                check_nonneg(ch)
                assert ch.lb >= rp["lb"]
                if ch.n >= 3:
                    r = ch.bound(1)
                    check_preservation(ch, inst, fixed=fx)
                    check_nonneg(ch)
                    assert r["lb"] >= par.lb and r["lb"] <= subtree_opt(inst, fx) * (1 + 1e-12) + 1e-9


@pytest.mark.parametrize("family", ["nug", "taib"])
def test_fold_of_fold_and_child_steps(orc, family):
    """Two warm levels (grandchild of a bounded child), preservation after every step."""
    inst = qapgen.make(family, 7, 3)
    par = orc.State(inst.F, inst.D)
    par.bound(1)
    ch = par.fold(2, 4)
    fx = child_fixed(par, (), 2, 4)
    ch.iteration0()
    check_preservation(ch, inst, fixed=fx)
    for name in STEPS:
        getattr(ch, name)()
        check_preservation(ch, inst, fixed=fx)
        check_nonneg(ch)
    g = ch.fold(0, 1)
    fg = child_fixed(ch, fx, 0, 1)
    check_preservation(g, inst, fixed=fg)
    r = g.bound(2)
    check_preservation(g, inst, fixed=fg)
    assert r["lb"] <= subtree_opt(inst, fg) + 1e-9


def test_constant_cost_child_is_exact(orc):
    """Every permutation costs the same: a warm child's bound is that cost."""
    c = qapgen.const(6, 2)
    opt = c.evaluate(list(range(6)))
    par = orc.State(c.F, c.D)
    par.bound(2)
    for a, b in [(0, 0), (3, 5), (5, 1)]:
        ch = par.fold(a, b)
        assert abs(ch.bound(2)["lb"] - opt) <= 1e-9 * opt


def test_fold_rejects_bad_arguments(orc):
    inst = qapgen.nug(4, 1)
    par = orc.State(inst.F, inst.D)
    par.bound(1)
    with pytest.raises(orc.OracleError):
        par.fold(4, 0)
    ch = par.fold(0, 0)          # n = 3
    with pytest.raises(orc.OracleError):
        ch.fold(0, 0)            # a child of size 2 is a leaf, not a state


@pytest.mark.parametrize("sb", [-1, 1])
@pytest.mark.parametrize("family,n", [("nug", 7), ("taib", 8), ("uniform", 8), ("nug", 9)])
def test_warm_bnb_optimum(orc, family, n, sb):
    inst = qapgen.make(family, n, 1)
    w = orc.bnb(inst.F, inst.D, T=2, sb_iters=sb, warm=True)
    assert w["opt"] == de.brute_force_opt(inst.F, inst.D)
    assert inst.evaluate(list(w["perm"])) == w["opt"]
    c = orc.bnb(inst.F, inst.D, T=2, sb_iters=sb)
    assert c["opt"] == w["opt"]
