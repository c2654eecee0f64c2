"""GPU: subtree-parallel B&B pieces through the C ABI.

* qap_bnb_frontier: the open nodes' bounds equal a fresh fix + bound of each node bit for bit;
  searching every frontier subtree (qap_bnb_run(root=...)) with the incumbent carried over
  gives the oracle B&B optimum.
* the scheduler (subtree.py) with 1, 2 and 3 workers (threads, each its own handle on
  cuda:0, a HashStore queue), with forced donations: optimum = brute force (n = 9) / the
  oracle B&B (n = 10); the permutation is optimal.
* the hooks: the sync callback sees every improvement; an abort from it surfaces as an error.
"""
import math
import threading

import numpy as np
import pytest

import qapgen
from tests import dualeval as de

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


@pytest.mark.parametrize("family,n,target", [("nug", 9, 4), ("taib", 10, 12), ("nug", 12, 30)])
def test_frontier_bounds_and_subtrees(orc, pkg, family, n, target):
    inst = qapgen.make(family, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D)
    nodes, fr = pkg.qap_bnb_frontier(h, 3, target, batch=4)
    assert len(nodes) >= target or fr["complete"] or len(nodes) > 0
    depths = {len(nd["fac"]) for nd in nodes}
    assert len(depths) == 1  # one BFS level
    h2 = pkg.qap_rlt2_create(n, inst.F, inst.D)
    for nd in nodes[:8]:
        pkg.qap_rlt2_fix(h2, list(zip(nd["fac"], nd["loc"])))
        assert pkg.qap_rlt2_bound(h2, 3)["lb"] == nd["lb"]
    # DFS order: lexicographic in the (facility, location) sequence of the minimal branching
    keys = [tuple(nd["loc"]) for nd in nodes]
    assert keys == sorted(keys)
    best = fr["opt"]
    for nd in nodes:
        r = pkg.qap_bnb_run(h, 3, UB0=math.inf if best < 0 else float(best), root=nd)
        if r["opt"] >= 0 and (best < 0 or r["opt"] < best):
            best = r["opt"]
    # reference: the one-worker DFS (pinned to the oracle B&B in test_gpu_parity) / brute force
    assert best == pkg.qap_bnb_solve(h2, 3)["opt"]
    if n <= 9:
        assert best == de.brute_force_opt(inst.F, inst.D)
    pkg.qap_destroy(h)
    pkg.qap_destroy(h2)


def test_frontier_exhausts_small_tree(orc, pkg):
    inst = qapgen.nug(7, 2)
    h = pkg.qap_rlt2_create(7, inst.F, inst.D)
    nodes, fr = pkg.qap_bnb_frontier(h, 2, 10 ** 6)
    assert nodes == [] and fr["complete"]
    assert fr["opt"] == de.brute_force_opt(inst.F, inst.D)
    assert inst.evaluate(list(fr["perm"])) == fr["opt"]
    pkg.qap_destroy(h)


@pytest.mark.parametrize("workers,sb", [(1, -1), (2, -1), (2, 1), (3, -1)])
def test_subtree_scheduler(orc, torch, pkg, workers, sb):
    import torch.distributed as dist
    from paper_1510_02065_b200 import subtree
    n = 9 if workers == 1 else 10
    inst = qapgen.nug(n, 1)
    store = dist.HashStore()
    hs = [pkg.qap_rlt2_create(n, inst.F, inst.D, stream=torch.cuda.Stream().cuda_stream) for _ in range(workers)]
    out = [None] * workers
    errs = []

    def body(r):
        try:
            # target=1: the frontier is the root alone, so other workers only get work by donation
            out[r] = subtree.subtree_bnb(pkg, hs[r], store, r, workers, 2, target=1, batch=2, sb_iters=sb,
                                         sync_every=1, prefix=f"w{workers}s{sb}/")
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(workers)]
    [t.start() for t in th]
    [t.join(300) for t in th]
    assert not errs, errs
    opt = de.brute_force_opt(inst.F, inst.D) if n <= 9 else orc.bnb(inst.F, inst.D, T=2)["opt"]
    for r in out:
        assert r["opt"] == opt
        assert inst.evaluate(r["perm"]) == opt
    if workers > 1:
        assert out[0]["donated"] > 0  # idle workers were fed by donation
        assert sum(w["tasks"] > 0 for w in out[0]["workers"]) >= 2
    for h in hs:
        pkg.qap_destroy(h)


def test_sync_hook_and_abort(pkg):
    inst = qapgen.nug(9, 3)
    h = pkg.qap_rlt2_create(9, inst.F, inst.D)
    seen = []

    def sync(best, perm):
        if best >= 0:
            assert inst.evaluate(list(perm)) == best
        seen.append(best)
        return -1, 0

    r = pkg.qap_bnb_run(h, 2, sync=sync, sync_every=1)
    assert seen[-1] == r["opt"] == de.brute_force_opt(inst.F, inst.D)
    found = [x for x in seen if x >= 0]
    assert all(a >= b for a, b in zip(found, found[1:]))  # incumbents only improve

    def bad(best, perm):
        raise KeyError("stop")

    with pytest.raises(KeyError):
        pkg.qap_bnb_run(h, 2, sync=bad)
    # a global incumbent from elsewhere prunes: with the optimum known up front nothing beats it
    r2 = pkg.qap_bnb_run(h, 2, sync=lambda b, p: (r["opt"], 0), sync_every=1)
    assert r2["bounded"] <= r["bounded"]
    pkg.qap_destroy(h)
