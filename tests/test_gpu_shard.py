"""Sharded bound on one GPU through an in-process group of G shards:
LB trace, B, C and the assembled D must equal the single-GPU bound bit for bit (the
per-element operations are identical; only where they run changes)."""
import numpy as np
import pytest

import qapgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    from paper_1510_02065_b200 import build
    build.build()
    import paper_1510_02065_b200 as p
    p.load_library()
    return p


@pytest.mark.parametrize("family,n,G,T", [("nug", 8, 2, 4), ("taib", 9, 3, 3), ("uniform", 12, 2, 3),
                                          ("nug", 12, 4, 2), ("taib", 14, 3, 2), ("nug", 10, 8, 2)])
def test_group_equals_single(pkg, family, n, G, T):
    inst = qapgen.make(family, n, 3)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D)
    ref = pkg.qap_rlt2_bound(h, T, trace=True)
    B1, C1, D1, lb1 = pkg.qap_rlt2_dual_copy(h)
    pkg.qap_destroy(h)
    grp = pkg.Group(G, n, inst.F, inst.D)
    outs = grp.bound(T, trace=True)
    for o in outs:
        assert o["lb_glb"] == ref["lb_glb"]
        assert (o["trace"] == ref["trace"]).all()
    B, C, D, lb = grp.dual()
    assert lb == lb1
    assert (B == B1).all() and (C == C1).all()
    assert (D == D1).all()
    for hh in grp.handles[1:]:
        Bq, Cq, _, lbq = pkg.qap_rlt2_dual_copy(hh, want_D=False)
        assert (Bq == B1).all() and (Cq == C1).all() and lbq == lb1
    info = [pkg.qap_rlt2_shard_info(hh) for hh in grp.handles]
    assert sum(i["blk_hi"] - i["blk_lo"] for i in info) == n * n * (n - 1) * (n - 1) // 2
    grp.close()


def test_group_fixed_node_and_stop(pkg):
    inst = qapgen.taib(11, 2)
    fixed = ((3, 5), (0, 1))
    h = pkg.qap_rlt2_create(11, inst.F, inst.D)
    pkg.qap_rlt2_fix(h, fixed)
    ref = pkg.qap_rlt2_bound(h, 30, K=1e-3, UB=1e9, trace=True)
    pkg.qap_destroy(h)
    grp = pkg.Group(3, 11, inst.F, inst.D)
    grp.fix(fixed)
    outs = grp.bound(30, K=1e-3, UB=1e9, trace=True)
    for o in outs:
        assert (o["iters"], o["status"]) == (ref["iters"], ref["status"])
        assert (o["trace"] == ref["trace"]).all()
    grp.close()


def test_group_n30_one_iteration(pkg):
    inst = qapgen.nug(30, 1)
    h = pkg.qap_rlt2_create(30, inst.F, inst.D)
    ref = pkg.qap_rlt2_bound(h, 1)
    pkg.qap_destroy(h)
    grp = pkg.Group(2, 30, inst.F, inst.D)
    outs = grp.bound(1)
    assert all(o["lb"] == ref["lb"] for o in outs)
    grp.close()


def test_nccl_loadable(pkg):
    """The NCCL transport resolves libnccl (torch's copy) and creates a unique id."""
    import torch.distributed  # noqa: F401  (torch's NCCL is loaded with torch)
    uid = pkg.qap_nccl_unique_id()
    assert len(uid) == 128 and any(uid)
