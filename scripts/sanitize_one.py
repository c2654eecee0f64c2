"""Small workloads for compute-sanitizer: bounds at N=8 and 12 (+ fixed node), a LAP
batch with m = 28 and 38, an in-process sharded group, the TMA transfer (n = 11, 12), warm
fold + bound, warm and strong-branching B&B."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1510_02065_b200 as pkg
import qapgen

torch.cuda.set_device(0)
for n, fam in ((8, "nug"), (12, "taib")):
    inst = qapgen.make(fam, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=pkg.QAP_FLAG_NO_GRAPH)
    print(n, pkg.qap_rlt2_bound(h, 3)["lb"])
    pkg.qap_rlt2_fix(h, ((0, 1), (2, 3)))
    print(n, pkg.qap_rlt2_bound(h, 2)["lb"])
    pkg.qap_destroy(h)
for m in (28, 38):
    M = torch.from_numpy(np.stack([qapgen.random_matrix(m, s, "real") for s in range(64)])).cuda()
    S = torch.zeros(64, dtype=torch.float64, device="cuda")
    pkg.qap_lap_batch(M, M, S)
    torch.cuda.synchronize()
    print(m, S.sum().item())
inst = qapgen.nug(9, 2)
g = pkg.Group(3, 9, inst.F, inst.D, flags=pkg.QAP_FLAG_NO_GRAPH)
print("group", g.bound(2)[0]["lb"])
g.close()
# TMA transfer (n >= 10, even and odd n - 2), warm fold + bound, warm B&B, strong branching
for n, fam in ((11, "taib"), (12, "nug")):
    inst = qapgen.make(fam, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=pkg.QAP_FLAG_NO_GRAPH)
    c = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=pkg.QAP_FLAG_NO_GRAPH)
    print("tma", n, pkg.qap_rlt2_bound(h, 3)["lb"])
    pkg.qap_rlt2_fold(c, h, 0, 2)
    print("fold", n, pkg.qap_rlt2_bound(c, 2)["lb"])
    pkg.qap_destroy(c)
    pkg.qap_destroy(h)
inst = qapgen.nug(9, 1)
h = pkg.qap_rlt2_create(9, inst.F, inst.D, flags=pkg.QAP_FLAG_NO_GRAPH)
print("warm bnb", pkg.qap_bnb_solve(h, 2, batch=3, warm=True)["opt"])
print("sb bnb", pkg.qap_bnb_solve(h, 2, batch=3, sb_iters=1)["opt"])
pkg.qap_destroy(h)
