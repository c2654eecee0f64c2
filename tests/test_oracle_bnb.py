"""Pins of the oracle's minimal B&B (SURVEY §8(b) caller): the optimum
equals brute-force enumeration and the returned permutation attains it."""
import math

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
