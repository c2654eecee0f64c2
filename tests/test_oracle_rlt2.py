"""Pins of the oracle's RLT2 dual ascent against what the paper and
the mathematics fix: preservation of every permutation's cost, nonnegativity
(P:163), the Gilmore–Lawler bound at iteration 0 (closed form), LB <= brute-force OPT,
monotone LB (each LB' >= 0), constant-cost instances (LB = OPT exactly), the zero
instance, class-sum conservation of the transfer and SPEC worked examples."""
import json
import math
import os

import numpy as np
import pytest

import qapgen
from tests import dualeval as de

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def check_preservation(st, inst, perms_full=None, fixed=()):
    n = st.n
    perms, val = de.dual_values(n, st.lb, st.B, st.C, st.D)
    I, J = st.free_maps()
    full = np.zeros((len(perms), inst.n), dtype=np.int64)
    for a, b in fixed:
        full[:, a] = b
    for x in range(n):
        full[:, I[x]] = J[perms[:, x]]
    cost = de.full_costs(inst.F, inst.D, full)
    err = np.abs(val - cost).max() / max(1.0, float(np.abs(cost).max()))
    assert err <= 1e-12, f"preservation error {err}"


def check_nonneg(st):
    for X in (st.B, st.C, st.D):
        assert (X >= 0).all()
        assert not np.signbit(X).any()


STEPS = ["spread_b", "spread_c_transfer_d", "concentrate_d", "transfer_c", "concentrate_c", "concentrate_b"]


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
@pytest.mark.parametrize("n", [4, 5, 6])
def test_preservation_every_prefix(orc, family, n):
    """after ANY prefix of the operation sequence every permutation's cost is
    unchanged; every stored entry stays >= 0."""
    for seed in range(1, 4 if n == 6 else 6):
        inst = qapgen.make(family, n, seed)
        st = orc.State(inst.F, inst.D)
        check_preservation(st, inst)
        st.iteration0()
        check_preservation(st, inst)
        check_nonneg(st)
        for _ in range(2):
            for name in STEPS:
                getattr(st, name)()
                check_preservation(st, inst)
                check_nonneg(st)


@pytest.mark.parametrize("family", ["taib", "uniform"])   # uniform: asymmetric F and D
@pytest.mark.parametrize("fixed", [((0, 2),), ((1, 0), (4, 3)), ((6, 6), (2, 5), (0, 1))])
def test_preservation_fixed_nodes(orc, family, fixed):
    """O0 reduction (cold child): kappa + reduced dual objective = full cost of every completion."""
    inst = qapgen.make(family, 9 if len(fixed) == 3 else 8, 2)
    st = orc.State(inst.F, inst.D, fixed)
    assert st.n == inst.n - len(fixed)
    check_preservation(st, inst, fixed=fixed)
    st.bound(2)
    check_preservation(st, inst, fixed=fixed)
    check_nonneg(st)


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
@pytest.mark.parametrize("n", [4, 6, 8, 12, 20])
def test_iteration0_is_gilmore_lawler(orc, family, n):
    """Reading R1: iteration 0 (concentrate C->B->LB from the initial costs) equals the
    Gilmore–Lawler bound computed from its textbook definition."""
    for seed in (1, 2):
        inst = qapgen.make(family, n, seed)
        out = orc.bound(inst.F, inst.D, T=0)
        assert out["lb_glb"] == de.gilmore_lawler(inst.F, inst.D)
        assert out["lb"] == out["lb_glb"]


def test_iteration0_gl_fixed(orc):
    inst = qapgen.nug(12, 3)
    for fixed in [((0, 5),), ((3, 3), (7, 0))]:
        st = orc.State(inst.F, inst.D, fixed)
        out = st.bound(0)
        assert out["lb_glb"] == de.gilmore_lawler(inst.F, inst.D, fixed)


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
@pytest.mark.parametrize("n", [5, 6, 7, 8])
def test_bound_valid_and_monotone(orc, family, n):
    """LB <= brute-force OPT (P:169 validity), LB nondecreasing (LB' = LAP value >= 0),
    LB >= GLB."""
    for seed in range(1, 4):
        inst = qapgen.make(family, n, seed)
        opt = de.brute_force_opt(inst.F, inst.D)
        out = orc.bound(inst.F, inst.D, T=8, trace=True)
        tr = np.concatenate([[out["lb_glb"]], out["trace"]])
        assert (np.diff(tr) >= 0).all()
        assert out["lb"] <= opt * (1 + 1e-12) + 1e-9
        assert out["lb"] >= out["lb_glb"]


@pytest.mark.slow
def test_bound_valid_n9(orc):
    for family in ("nug", "taib"):
        inst = qapgen.make(family, 9, 1)
        opt = de.brute_force_opt(inst.F, inst.D)
        out = orc.bound(inst.F, inst.D, T=5)
        assert out["lb"] <= opt * (1 + 1e-12) + 1e-9


@pytest.mark.parametrize("n", [4, 6, 9, 12])
def test_constant_cost_instance(orc, n):
    """Every permutation costs the same when f_ik = 1 (i != k): GLB = OPT exactly and
    every later LB' = 0."""
    inst = qapgen.const(n, 3)
    opt = inst.evaluate(list(range(n)))
    st = orc.State(inst.F, inst.D)
    out = st.bound(3, trace=True)
    assert out["lb_glb"] == opt
    assert (out["trace"] == opt).all()


def test_zero_instance(orc):
    inst = qapgen.zero(6)
    out = orc.bound(inst.F, inst.D, T=3)
    assert out["lb"] == 0.0 and out["lb_glb"] == 0.0


def test_c_pairs_equal_after_concentrate_d(orc):
    """After D->C concentration c_ij[kl] == c_kl[ij] exactly, so the C transfer (P:189,
    reading R13) is an exact no-op."""
    inst = qapgen.taib(7, 4)
    st = orc.State(inst.F, inst.D)
    st.iteration0()
    st.spread_b()
    st.spread_c_transfer_d()
    st.concentrate_d()
    C = st.C.copy()
    n = st.n
    for i in range(n):
        for j in range(n):
            for k in range(n):
                for l in range(n):
                    if i != k and j != l:
                        assert C[i, j, de.skip1(k, i), de.skip1(l, j)] == C[k, l, de.skip1(i, k), de.skip1(j, l)]
    st.transfer_c()
    assert (st.C == C).all()


def test_transfer_class_members_equal_and_conserved(orc):
    """the transfer is zero-sum within each class of 6 complementary coefficients
    (3 stored members), and with the mean policy (reading R11) leaves the 3 members equal."""
    inst = qapgen.uniform(6, 5)
    st = orc.State(inst.F, inst.D)
    st.iteration0()
    st.spread_b()
    st.spread_c_transfer_d()
    st.concentrate_d()
    st.concentrate_c()
    st.concentrate_b()
    st.spread_b()
    n = st.n
    bidx = de.block_index(n)
    C = st.C.copy()
    D0 = st.D.copy()
    sig = {}
    for (i, j, k, l), t in bidx.items():
        sig[t] = (C[i, j, de.skip1(k, i), de.skip1(l, j)] + C[k, l, de.skip1(i, k), de.skip1(j, l)]) / (2 * (n - 2))
    st.spread_c_transfer_d()
    D1 = st.D
    for i in range(n):
        for k in range(i + 1, n):
            for p in range(k + 1, n):
                for j in range(n):
                    for l in range(n):
                        for q in range(n):
                            if len({j, l, q}) < 3:
                                continue
                            mem = [(bidx[(i, j, k, l)], de.skip2(p, i, k), de.skip2(q, j, l)),
                                   (bidx[(i, j, p, q)], de.skip2(k, i, p), de.skip2(l, j, q)),
                                   (bidx[(k, l, p, q)], de.skip2(i, k, p), de.skip2(j, l, q))]
                            before = sum(D0[b, r, c] + sig[b] for b, r, c in mem)
                            after = [D1[b, r, c] for b, r, c in mem]
                            assert after[0] == after[1] == after[2]
                            assert abs(sum(after) - before) <= 1e-12 * max(1.0, before)
    assert (st.C == 0).all()


def test_transfer_idempotent(orc):
    """SPEC P6: applying the transfer again with nothing spread changes nothing
    (up to the rounding of ((a+a)+a)/3)."""
    inst = qapgen.nug(7, 2)
    st = orc.State(inst.F, inst.D)
    st.bound(1)
    st.spread_b()
    st.spread_c_transfer_d()
    D1 = st.D.copy()
    st.spread_c_transfer_d()        # C is zero now: sigma = 0
    assert np.allclose(st.D, D1, rtol=4e-16, atol=0)


# --- worked examples (tests/golden/spec_examples.json) ---------------------------

def _zero_state(orc, n):
    z = np.zeros((n, n), np.int64)
    st = orc.State(z, z)
    st._L.oracle_iteration0(st._h)   # mark non-fresh; all zero anyway
    return st


def test_example_spread_b(orc):
    g = GOLDEN["spread_b"]
    st = _zero_state(orc, g["n"])
    i, j, val = g["b"]
    st.B[i, j] = val
    st.spread_b()
    assert (st.C[i, j] == g["c_after"]).all()
    assert st.B[i, j] == 0
    others = np.ones(st.C.shape[:2], bool)
    others[i, j] = False
    assert (st.C[others] == 0).all()


def test_example_spread_c(orc):
    g = GOLDEN["spread_c"]
    n = g["n"]
    st = _zero_state(orc, n)
    for i, j, k, l, val in g["c"]:
        st.C[i, j, de.skip1(k, i), de.skip1(l, j)] = val
    st.spread_c_transfer_d()
    bidx = de.block_index(n)
    blk = st.D[bidx[(0, 1, 2, 3)]]
    assert (blk == g["after_transfer"]).all()
    assert abs(st.D.sum() - g["spread"] * (n - 2) ** 2) < 1e-12
    assert (st.C == 0).all()


def test_example_transfer_triple(orc):
    g = GOLDEN["transfer_d"]
    n = 4
    st = _zero_state(orc, n)
    bidx = de.block_index(n)
    # class {(0,0),(1,1),(2,2)}: members e1, e2, e3
    mem = [(bidx[(0, 0, 1, 1)], de.skip2(2, 0, 1), de.skip2(2, 0, 1)),
           (bidx[(0, 0, 2, 2)], de.skip2(1, 0, 2), de.skip2(1, 0, 2)),
           (bidx[(1, 1, 2, 2)], de.skip2(0, 1, 2), de.skip2(0, 1, 2))]
    for (b, r, c), val in zip(mem, g["values"]):
        st.D[b, r, c] = val
    st.spread_c_transfer_d()
    for b, r, c in mem:
        assert st.D[b, r, c] == g["after"]


def test_example_concentrate_d(orc):
    g = GOLDEN["concentrate_d"]
    n = g["n"]
    st = _zero_state(orc, n)
    i, j, k, l = g["block"]
    bidx = de.block_index(n)
    st.D[bidx[(i, j, k, l)]] = np.array(g["M"], float)
    st.concentrate_d()
    assert st.C[i, j, de.skip1(k, i), de.skip1(l, j)] == g["S"]
    assert st.C[k, l, de.skip1(i, k), de.skip1(j, l)] == g["S"]
    assert st.C.sum() == 2 * g["S"]


def test_example_concentrate_c(orc):
    g = GOLDEN["concentrate_c"]
    st = _zero_state(orc, g["n"])
    st.C[0, 0] = np.array(g["M"], float)
    st.concentrate_c()
    assert st.B[0, 0] == g["S"]


def test_example_concentrate_b(orc):
    g = GOLDEN["concentrate_b"]
    st = _zero_state(orc, g["n"])
    st.B[:] = 1.0
    assert st.concentrate_b() == g["S"]


def test_stop_rules(orc):
    """Readings R14/R15: prune when LB > UB - 1 + 1e-6; converge when LB'/UB < K."""
    inst = qapgen.nug(8, 1)
    opt = de.brute_force_opt(inst.F, inst.D)
    glb = orc.bound(inst.F, inst.D, T=0)["lb"]
    out = orc.bound(inst.F, inst.D, T=50, UB=math.floor(glb))      # GLB already prunes
    assert out["status"] == 2 and out["iters"] == 0
    out = orc.bound(inst.F, inst.D, T=50, K=1.0, UB=opt)           # LB' / UB < 1 at once
    assert out["status"] in (1, 2) and out["iters"] == 1
    out = orc.bound(inst.F, inst.D, T=3, UB=math.inf)
    assert out["status"] == 0 and out["iters"] == 3


# --- the RLT1 ascent's C pair mean ---------------------

RLT1_STEPS = ["spread_b", "transfer_c", "concentrate_c", "concentrate_b"]


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
@pytest.mark.parametrize("n", [4, 5, 6])
def test_rlt1_preservation_every_prefix(orc, family, n):
    """P:169 for the RLT1 step sequence (Algorithm 1 without the D operations):
    after every prefix of spread B->C, C pair mean, C->B, B->LB every permutation's cost is
    unchanged and every entry stays >= 0.  A pair 'mean' with a wrong divisor or a
    one-sided write breaks the evaluation of the permutations using the pair."""
    for seed in range(1, 4 if n == 6 else 6):
        inst = qapgen.make(family, n, seed)
        st = orc.State(inst.F, inst.D)
        st.iteration0()
        for _ in range(3):
            for name in RLT1_STEPS:
                getattr(st, name)()
                check_preservation(st, inst)
                check_nonneg(st)


def test_transfer_c_pairs_equal_and_conserved(orc):
    """P:222-223 (zero-sum) with reading R13 (mean): after the C transfer each complementary
    pair c_ij[kl], c_kl[ij] is equal and keeps its sum, on a state where the pairs differ
    (after spreading B -> C in the RLT1 sequence)."""
    inst = qapgen.uniform(7, 3)
    st = orc.State(inst.F, inst.D)
    st.iteration0()
    st.spread_b()
    C0 = st.C.copy()
    st.transfer_c()
    C1 = st.C
    n = st.n
    differ = 0
    for i in range(n):
        for j in range(n):
            for k in range(i + 1, n):
                for l in range(n):
                    if l == j:
                        continue
                    a = (i, j, de.skip1(k, i), de.skip1(l, j))
                    b = (k, l, de.skip1(i, k), de.skip1(j, l))
                    differ += C0[a] != C0[b]
                    assert C1[a] == C1[b]
                    assert abs((C1[a] + C1[b]) - (C0[a] + C0[b])) <= 1e-15 * max(1.0, C0[a] + C0[b])
    assert differ > 0


def test_example_transfer_c(orc):
    """c_0123 = 4, c_2301 = 2 -> both 3; every other coefficient stays 0."""
    g = GOLDEN["transfer_c"]
    n = g["n"]
    st = _zero_state(orc, n)
    for i, j, k, l, val in g["c"]:
        st.C[i, j, de.skip1(k, i), de.skip1(l, j)] = val
    st.transfer_c()
    for i, j, k, l, _ in g["c"]:
        assert st.C[i, j, de.skip1(k, i), de.skip1(l, j)] == g["after"]
    assert st.C.sum() == 2 * g["after"]


@pytest.mark.parametrize("family", ["nug", "taib", "uniform"])
def test_rlt1_ascent_is_driven_by_the_pair_mean(orc, family):
    """Why the C transfer is in the RLT1 loop: without it an RLT1 iteration is
    stationary — spreading b_ij over a residual C_ij whose LAP value is 0 and concentrating
    it again returns b_ij, and B is a residual with LAP value 0, so LB' = 0 up to rounding.
    With the pair mean the ascent rises strictly above the Gilmore–Lawler bound (and stays
    <= the brute-force optimum) on instances where GLB < OPT."""
    for seed in (1, 2, 3):
        inst = qapgen.make(family, 7, seed)
        opt = de.brute_force_opt(inst.F, inst.D)
        glb = de.gilmore_lawler(inst.F, inst.D)
        assert glb < opt
        st = orc.State(inst.F, inst.D)
        st.iteration0()
        for _ in range(3):                       # the sequence WITHOUT the pair mean
            st.spread_b()
            st.concentrate_c()
            lbp = st.concentrate_b()
            assert lbp <= 1e-9 * max(1.0, glb)
        st = orc.State(inst.F, inst.D)
        lb = st.rlt1_bound(3)
        assert lb > glb + 1e-6 * max(1.0, glb), (family, seed, lb, glb)
        assert lb <= opt * (1 + 1e-12) + 1e-9


def test_all_cores_mode_is_bit_identical(orc):
    """SURVEY §8(d) oracle timing mode (ii): the OpenMP loops over independent units (blocks,
    classes, pairs) give the same bits as the sequential oracle."""
    inst = qapgen.taib(12, 2)
    ref = orc.State(inst.F, inst.D)
    r1 = ref.bound(3, trace=True)
    try:
        orc.set_threads(4)
        st = orc.State(inst.F, inst.D)
        r4 = st.bound(3, trace=True)
    finally:
        orc.set_threads(1)
    assert (r1["trace"] == r4["trace"]).all() and r1["lb"] == r4["lb"]
    for a, b in ((ref.B, st.B), (ref.C, st.C), (ref.D, st.D)):
        assert a.tobytes() == b.tobytes()
