"""GPU parity of the warm child (qap_rlt2_fold, R31)
against the oracle's fold (tests/test_oracle_warm.py pins it): the folded B, C, D and LB
are bit-identical, and so is everything the child's own bound does afterwards — from
bounded parents, fresh parents (D lazily zero), parents with fixed pairs and over two warm
levels.  Argument and state errors surface as QapError."""
import numpy as np
import pytest

import qapgen
from tests.test_gpu_parity import compare_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    t.cuda.set_device(0)
    return t


@pytest.fixture(scope="module")
def pkg(torch):
    import paper_1510_02065_b200 as p
    return p


CASES = [("nug", 6, (), 2), ("taib", 8, (), 2), ("uniform", 8, ((1, 3),), 1), ("nug", 12, (), 2),
         ("taib", 12, ((0, 5), (4, 1)), 1), ("nug", 9, (), 0), ("nug", 9, (), -1)]


@pytest.mark.parametrize("family,n,fixed,T1", CASES)
def test_fold_then_bound_exact(orc, pkg, family, n, fixed, T1):
    """T1 = -1: the parent was only fixed (fresh: initial B, C; D lazily zero)."""
    inst = qapgen.make(family, n, 1)
    hp = pkg.qap_rlt2_create(n, inst.F, inst.D)
    hc = pkg.qap_rlt2_create(n, inst.F, inst.D)
    pkg.qap_rlt2_fix(hp, list(fixed))
    sp = orc.State(inst.F, inst.D, fixed)
    if T1 >= 0:
        g = pkg.qap_rlt2_bound(hp, T1)
        o = sp.bound(T1)
        assert g["lb"] == o["lb"]
    I, J = sp.free_maps()
    m = len(I)
    picks = sorted({(0, 0), (m - 1, m - 1), (1, m - 2), (m // 2, 1)})
    for a, b in picks:
        pkg.qap_rlt2_fold(hc, hp, int(I[a]), int(J[b]))
        sc = sp.fold(a, b)
        compare_state(pkg, hc, sc)
        g = pkg.qap_rlt2_bound(hc, 2, trace=True)
        o = sc.bound(2, trace=True)
        assert g["lb"] == o["lb"] and g["lb_glb"] == o["lb_glb"]
        assert (g["trace"] == o["trace"]).all()
        compare_state(pkg, hc, sc)
    pkg.qap_destroy(hp)
    pkg.qap_destroy(hc)


def test_two_warm_levels(orc, pkg):
    inst = qapgen.taib(11, 2)
    h = [pkg.qap_rlt2_create(11, inst.F, inst.D) for _ in range(3)]
    s0 = orc.State(inst.F, inst.D)
    pkg.qap_rlt2_bound(h[0], 2)
    s0.bound(2)
    pkg.qap_rlt2_fold(h[1], h[0], 3, 7)
    I, J = s0.free_maps()
    s1 = s0.fold(int(np.where(I == 3)[0][0]), int(np.where(J == 7)[0][0]))
    assert pkg.qap_rlt2_bound(h[1], 3)["lb"] == s1.bound(3)["lb"]
    pkg.qap_rlt2_fold(h[2], h[1], 0, 0)
    I1, J1 = s1.free_maps()
    s2 = s1.fold(int(np.where(I1 == 0)[0][0]), int(np.where(J1 == 0)[0][0]))
    compare_state(pkg, h[2], s2)
    assert pkg.qap_rlt2_bound(h[2], 2)["lb"] == s2.bound(2)["lb"]
    compare_state(pkg, h[2], s2)
    # the parent is untouched by folding its children: it continues exactly like the oracle
    assert pkg.qap_rlt2_bound(h[1], 1)["lb"] == s1.bound(1)["lb"]
    for x in h:
        pkg.qap_destroy(x)


def test_fold_errors(pkg):
    inst = qapgen.nug(8, 1)
    hp = pkg.qap_rlt2_create(8, inst.F, inst.D)
    hc = pkg.qap_rlt2_create(8, inst.F, inst.D)
    pkg.qap_rlt2_fix(hp, [(0, 0)])
    with pytest.raises(pkg.QapError):
        pkg.qap_rlt2_fold(hc, hp, 0, 3)          # facility 0 already fixed
    with pytest.raises(pkg.QapError):
        pkg.qap_rlt2_fold(hc, hp, 8, 3)          # out of range
    other = qapgen.taib(8, 1)
    ho = pkg.qap_rlt2_create(8, other.F, other.D)
    with pytest.raises(pkg.QapError):
        pkg.qap_rlt2_fold(ho, hp, 1, 1)          # another instance
    pkg.qap_rlt2_step(hp, pkg.PHASE_ITER0)
    pkg.qap_rlt2_step(hp, pkg.PHASE_TRANSFER)
    with pytest.raises(pkg.QapError):
        pkg.qap_rlt2_fold(hc, hp, 1, 1)          # parent mid-iteration
    small = qapgen.nug(4, 1)
    h4 = pkg.qap_rlt2_create(4, small.F, small.D)
    h4c = pkg.qap_rlt2_create(4, small.F, small.D)
    pkg.qap_rlt2_fix(h4, [(0, 0)])
    with pytest.raises(pkg.QapError):
        pkg.qap_rlt2_fold(h4c, h4, 1, 1)         # child of size 2: a leaf
    for x in (hp, hc, ho, h4, h4c):
        pkg.qap_destroy(x)


@pytest.mark.parametrize("batch", [1, 4, 16])
@pytest.mark.parametrize("family,n,sb", [("nug", 7, -1), ("taib", 8, -1), ("uniform", 8, -1), ("nug", 10, -1),
                                         ("nug", 9, 1), ("taib", 9, 1)])
def test_warm_bnb_parity(orc, pkg, family, n, sb, batch):
    """Warm B&B: node counts, optimum and permutation identical to the oracle's warm B&B
    (one node at a time) also with children bounded concurrently; optimum = brute force."""
    from tests import dualeval as de
    inst = qapgen.make(family, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D)
    g = pkg.qap_bnb_solve(h, 2, batch=batch, sb_iters=sb, warm=True)
    o = orc.bnb(inst.F, inst.D, T=2, sb_iters=sb, warm=True)
    assert g["opt"] == o["opt"]
    assert (g["perm"] == o["perm"]).all()
    assert (g["bounded"], g["leaves"], g["pruned"], g["sb_cut"]) == (o["bounded"], o["leaves"], o["pruned"],
                                                                     o["sb_cut"])
    if n <= 9:
        assert g["opt"] == de.brute_force_opt(inst.F, inst.D)
    # cold search on the same handle afterwards is unaffected
    c = pkg.qap_bnb_solve(h, 2, batch=batch, sb_iters=sb)
    oc = orc.bnb(inst.F, inst.D, T=2, sb_iters=sb)
    assert (c["bounded"], c["opt"]) == (oc["bounded"], oc["opt"])
    pkg.qap_destroy(h)


def test_warm_bnb_checkpoint_resume(orc, pkg, tmp_path):
    inst = qapgen.nug(10, 2)
    h = pkg.qap_rlt2_create(10, inst.F, inst.D)
    ref = pkg.qap_bnb_run(h, 2, batch=4, warm=True)
    path = str(tmp_path / "warm.ckpt")
    r = pkg.qap_bnb_run(h, 2, batch=4, warm=True, checkpoint_path=path, max_nodes=9)
    assert not r["complete"]
    while not r["complete"]:
        r = pkg.qap_bnb_run(h, 2, batch=3, warm=True, checkpoint_path=path, max_nodes=7, resume=True)
    assert (r["opt"], r["bounded"], r["leaves"], r["pruned"]) == (ref["opt"], ref["bounded"], ref["leaves"],
                                                                   ref["pruned"])
    with pytest.raises(pkg.QapError):  # a cold run cannot resume a warm checkpoint
        pkg.qap_bnb_run(h, 2, batch=4, checkpoint_path=path, resume=True)
    pkg.qap_destroy(h)


def test_warm_subtree_workers(orc, torch, pkg):
    import threading
    import torch.distributed as dist
    from paper_1510_02065_b200 import subtree
    from tests import dualeval as de
    inst = qapgen.taib(9, 3)
    store = dist.HashStore()
    hs = [pkg.qap_rlt2_create(9, inst.F, inst.D, stream=torch.cuda.Stream().cuda_stream) for _ in range(2)]
    out = [None, None]

    def body(r):
        out[r] = subtree.subtree_bnb(pkg, hs[r], store, r, 2, 2, target=1, batch=3, sync_every=1, warm=True,
                                     prefix="warm/")

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(300) for t in th]
    opt = de.brute_force_opt(inst.F, inst.D)
    assert out[0]["opt"] == out[1]["opt"] == opt
    assert inst.evaluate(out[0]["perm"]) == opt
    for x in hs:
        pkg.qap_destroy(x)
