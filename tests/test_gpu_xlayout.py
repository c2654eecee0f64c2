"""GPU: the class layout of the level-2 dual (QAP_FLAG_CLASS_LAYOUT, nodes with
n >= 16) runs the same per-class and per-block operations as the default stored-block
layout, so whole dual states are bit-identical between the two — after
bounds at the root and at fixed nodes, for even and odd n (odd n pads the innermost
stride), for one and two columns per lane (n - 2 > 32), phase by phase against the
oracle, across exports in the middle of an iteration, and for warm children folded from
a class-layout parent."""
import numpy as np
import pytest

import qapgen
from tests.test_gpu_parity import compare_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    import paper_1510_02065_b200 as p
    return p


def _state(pkg, n, inst, flags, fixed, T):
    h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=flags)
    pkg.qap_rlt2_fix(h, list(fixed))
    r = pkg.qap_rlt2_bound(h, T, trace=True)
    B, C, D, lb = pkg.qap_rlt2_dual_copy(h)
    pkg.qap_destroy(h)
    return r, B, C, D, lb


@pytest.mark.parametrize("family,n,fixed,T", [("nug", 16, (), 3), ("taib", 17, (), 3), ("nug", 18, ((2, 7),), 2),
                                              ("taib", 21, ((0, 20), (9, 3)), 2), ("nug", 30, (), 2),
                                              ("taib", 35, (), 1)])
def test_class_layout_equals_block_layout(pkg, family, n, fixed, T):
    inst = qapgen.make(family, n, 3)
    ra, Ba, Ca, Da, la = _state(pkg, n, inst, pkg.QAP_FLAG_CLASS_LAYOUT, fixed, T)
    rb, Bb, Cb, Db, lb_ = _state(pkg, n, inst, 0, fixed, T)
    assert la == lb_ and (ra["trace"] == rb["trace"]).all() and ra["lb_glb"] == rb["lb_glb"]
    assert (Ba == Bb).all() and (Ca == Cb).all() and np.array_equal(Da, Db)


@pytest.mark.parametrize("family,n", [("taib", 16), ("nug", 17)])
def test_phase_by_phase_class_layout(orc, pkg, family, n):
    """Every phase of Algorithm 1 in the class layout leaves the oracle's B, C,
    D, LB (each export converts the class layout to stored blocks)."""
    inst = qapgen.make(family, n, 2)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=pkg.QAP_FLAG_CLASS_LAYOUT)
    st = orc.State(inst.F, inst.D)
    pkg.qap_rlt2_step(h, pkg.PHASE_ITER0)
    st.iteration0()
    for _ in range(2):
        pkg.qap_rlt2_step(h, pkg.PHASE_TRANSFER)
        st.spread_b()
        st.spread_c_transfer_d()
        compare_state(pkg, h, st)
        pkg.qap_rlt2_step(h, pkg.PHASE_CONC_D)
        st.concentrate_d()
        compare_state(pkg, h, st)
        pkg.qap_rlt2_step(h, pkg.PHASE_CONC_C)
        st.transfer_c()
        st.concentrate_c()
        pkg.qap_rlt2_step(h, pkg.PHASE_CONC_B)
        st.concentrate_b()
        compare_state(pkg, h, st)
    # a bound continuing after exports picks the state up from the class layout again
    g = pkg.qap_rlt2_bound(h, 2, trace=True)
    o = st.bound(2, trace=True)
    assert g["lb"] == o["lb"] and (g["trace"] == o["trace"]).all()
    compare_state(pkg, h, st)
    pkg.qap_destroy(h)


def test_fold_from_class_layout_parent(orc, pkg):
    """A warm child (n = 16) folded from a bounded class-layout parent (n = 17), and its own
    bound (class layout again), equal the oracle bit for bit."""
    n = 17
    inst = qapgen.taib(n, 4)
    hp = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=pkg.QAP_FLAG_CLASS_LAYOUT)
    hc = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=pkg.QAP_FLAG_CLASS_LAYOUT)
    sp = orc.State(inst.F, inst.D)
    assert pkg.qap_rlt2_bound(hp, 2)["lb"] == sp.bound(2)["lb"]
    I, J = sp.free_maps()
    for a, b in [(0, 0), (16, 3)]:
        pkg.qap_rlt2_fold(hc, hp, int(I[a]), int(J[b]))
        sc = sp.fold(a, b)
        g = pkg.qap_rlt2_bound(hc, 2, trace=True)
        o = sc.bound(2, trace=True)
        assert g["lb"] == o["lb"] and (g["trace"] == o["trace"]).all()
        compare_state(pkg, hc, sc)
    pkg.qap_destroy(hp)
    pkg.qap_destroy(hc)


@pytest.mark.parametrize("family,n,fixed,T", [("nug", 16, (), 3), ("taib", 17, ((3, 3),), 2), ("nug", 24, (), 2),
                                              ("nug", 30, (), 2), ("taib", 33, (), 1)])
def test_fused_iteration_equals_separate_kernels(pkg, family, n, fixed, T):
    """QAP_FLAG_FUSED (transfer tiles and level-2 LAPs in one persistent kernel, LAPs gated
    by per-facility completion counters) leaves the same dual state bit for bit."""
    inst = qapgen.make(family, n, 5)
    ra, Ba, Ca, Da, la = _state(pkg, n, inst, 0, fixed, T)
    rb, Bb, Cb, Db, lb_ = _state(pkg, n, inst, pkg.QAP_FLAG_FUSED | pkg.QAP_FLAG_CLASS_LAYOUT, fixed, T)
    assert la == lb_ and (ra["trace"] == rb["trace"]).all()
    assert (Ba == Bb).all() and (Ca == Cb).all() and np.array_equal(Da, Db)


@pytest.mark.parametrize("warm", [False, True])
def test_bnb_with_class_layout_root(pkg, warm):
    """A B&B whose root (n = 16) is bounded in the class layout and whose children (n <= 15)
    in the block layout — cold children, or warm ones folded / copied from class-layout
    states — takes the same decisions as the block-layout search: optimum, permutation and
    node counts."""
    inst = qapgen.nug(16, 3)
    out = []
    for fl in (0, pkg.QAP_FLAG_CLASS_LAYOUT):
        h = pkg.qap_rlt2_create(16, inst.F, inst.D, flags=fl)
        r = pkg.qap_bnb_solve(h, 2, batch=4, warm=warm)
        out.append(r)
        pkg.qap_destroy(h)
    a, b = out
    assert a["opt"] == b["opt"] and (np.asarray(a["perm"]) == np.asarray(b["perm"])).all()
    assert a["bounded"] == b["bounded"] and a["leaves"] == b["leaves"]
