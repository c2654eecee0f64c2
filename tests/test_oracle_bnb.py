"""Pins of the oracle's minimal B&B (SURVEY §8(b) caller): the optimum
equals brute-force enumeration and the returned permutation attains it."""
import math

import numpy as np

import pytest

import qapgen
from tests import dualeval as de


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
@pytest.mark.parametrize("n", [4, 6, 7, 8])
def test_bnb_optimum_is_bruteforce(orc, family, n):
    for seed in (1, 2):
        inst = qapgen.make(family, n, seed)
        opt = de.brute_force_opt(inst.F, inst.D)
        out = orc.bnb(inst.F, inst.D, T=2)
        assert out["opt"] == opt
        assert inst.evaluate(out["perm"]) == opt
        assert out["bounded"] >= 1 or n <= 3


def test_bnb_more_iterations_fewer_nodes(orc):
    inst = qapgen.nug(8, 1)
    a = orc.bnb(inst.F, inst.D, T=0)
    b = orc.bnb(inst.F, inst.D, T=3)
    assert a["opt"] == b["opt"]
    assert b["bounded"] + b["leaves"] <= a["bounded"] + a["leaves"]


def test_bnb_ub0_tight_prunes_root(orc):
    inst = qapgen.nug(7, 2)
    opt = de.brute_force_opt(inst.F, inst.D)
    out = orc.bnb(inst.F, inst.D, T=2, UB0=float(opt))
    # UB0 = OPT: nothing strictly better exists; every bounded node with LB > OPT-1 is cut
    assert out["opt"] in (-1, opt)


# --- RLT1 dual and strong branching ----------------------

@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
def test_rlt1_bound_valid_monotone(orc, family):
    """RLT1 ascent (Algorithm 1 without the D operations): every LB' >= 0 (monotone), LB <=
    brute-force OPT, iteration 0 = Gilmore–Lawler."""
    inst = qapgen.make(family, 7, 2)
    opt = de.brute_force_opt(inst.F, inst.D)
    st = orc.State(inst.F, inst.D)
    lb0 = st.rlt1_bound(0)
    assert lb0 == de.gilmore_lawler(inst.F, inst.D)
    prev = lb0
    for _ in range(6):
        lbp = st.rlt1_iteration()
        assert lbp >= 0.0
        assert st.lb >= prev
        prev = st.lb
    assert st.lb <= opt * (1 + 1e-12) + 1e-9


def test_rlt1_constant_cost(orc):
    inst = qapgen.const(8, 1)
    opt = inst.evaluate(list(range(8)))
    st = orc.State(inst.F, inst.D)
    assert st.rlt1_bound(4) == opt


@pytest.mark.parametrize("fixed", [(), ((2, 3),)])
def test_strong_branch_estimates_and_selection(orc, fixed):
    """Every estimate is a valid bound of its child (<= the child's brute-force optimum);
    the selected line maximises the min-estimate (ties: lowest index, rows first)."""
    inst = qapgen.taib(7, 3)
    est, kind, index = orc.strong_branch(inst.F, inst.D, fixed, T=2)
    n = inst.n - len(fixed)
    ff = {a for a, _ in fixed}
    fl = {b for _, b in fixed}
    I = [x for x in range(inst.n) if x not in ff]
    J = [x for x in range(inst.n) if x not in fl]
    import itertools
    for a in range(n):
        for b in range(n):
            child = dict(fixed)
            child[I[a]] = J[b]
            # brute-force optimum of the child's completions
            rest_f = [x for x in range(inst.n) if x not in child]
            rest_l = [x for x in range(inst.n) if x not in child.values()]
            best = min(inst.evaluate([{**child, **dict(zip(rest_f, pl))}[x] for x in range(inst.n)])
                       for pl in itertools.permutations(rest_l))
            assert est[a, b] <= best * (1 + 1e-12) + 1e-9
            # an independent State gives the same estimate
            st = orc.State(inst.F, inst.D, tuple(child.items()))
            assert st.rlt1_bound(2) == est[a, b]
    rows, cols = est.min(axis=1), est.min(axis=0)
    best = max(rows.max(), cols.max())
    exp = (0, int(np.argmax(rows))) if rows.max() >= cols.max() else (1, int(np.argmax(cols)))
    assert (kind, index) == exp and max(rows[index] if kind == 0 else cols[index], best) == best


@pytest.mark.parametrize("family,n", [("nug", 7), ("taib", 8), ("uniform", 7)])
def test_bnb_strong_branching_optimum(orc, family, n):
    inst = qapgen.make(family, n, 1)
    opt = de.brute_force_opt(inst.F, inst.D)
    out = orc.bnb(inst.F, inst.D, T=2, sb_iters=1)
    assert out["opt"] == opt and inst.evaluate(out["perm"]) == opt
    plain = orc.bnb(inst.F, inst.D, T=2)
    assert plain["opt"] == opt


# --- BASELINE config 2 (nug12-shaped, seed 1): oracle B&B vs brute force -------------------

def _golden_n12():
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "n12_nug_seed1_bnb.json")))


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
def test_qap_bruteforce_matches_enumeration(orc, family):
    """The C enumerator behind the N = 12 golden optimum agrees with the vectorised numpy
    enumeration (tests/dualeval.py) and its permutation attains the optimum."""
    for n in (5, 7, 8):
        inst = qapgen.make(family, n, 3)
        opt, perm = orc.qap_bruteforce(inst.F, inst.D)
        assert opt == de.brute_force_opt(inst.F, inst.D)
        assert inst.evaluate([int(x) for x in perm]) == opt


def test_bnb_config2_n12_optimum_is_bruteforce(orc):
    """BASELINE config 2: the oracle B&B with T = 10 (cold children) solves the nug12-shaped
    instance to the brute-force optimum over all 12! permutations (committed by
    scripts/golden_bnb_n12.py), with the committed node counts."""
    g = _golden_n12()
    inst = qapgen.nug(g["N"], 1)
    o = orc.bnb(inst.F, inst.D, T=g["T"])
    assert o["opt"] == g["bruteforce"]["opt"]
    assert inst.evaluate([int(x) for x in o["perm"]]) == g["bruteforce"]["opt"]
    c = g["bnb"]["cold"]
    assert (o["bounded"], o["leaves"], o["pruned"]) == (c["bounded"], c["leaves"], c["pruned"])
    assert list(o["perm"]) == c["perm"]
