"""Small workloads for compute-sanitizer: bounds at N=8 and 12 (+ fixed node), a LAP
batch with m = 28 and 38, and an in-process sharded group."""
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
