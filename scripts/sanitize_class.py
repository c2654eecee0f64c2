"""Small class-layout workloads for compute-sanitizer (QAP_FLAG_CLASS_LAYOUT, n = 16, 17):
k_transfer_x, the level-2 LAP with TMA gather4/scatter4, both layout conversions (export,
warm fold from a class-layout parent), and the experimental fused kernel."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1510_02065_b200 as pkg
import qapgen

torch.cuda.set_device(0)
CL = pkg.QAP_FLAG_CLASS_LAYOUT | pkg.QAP_FLAG_NO_GRAPH
for n, fam in ((16, "nug"), (17, "taib")):
    inst = qapgen.make(fam, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=CL)
    c = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=CL)
    print("class", n, pkg.qap_rlt2_bound(h, 2)["lb"])
    B, C, D, lb = pkg.qap_rlt2_dual_copy(h)
    pkg.qap_rlt2_fold(c, h, 0, 2)
    print("fold", n, pkg.qap_rlt2_bound(c, 1)["lb"])
    pkg.qap_destroy(c)
    pkg.qap_destroy(h)
    f = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=CL | pkg.QAP_FLAG_FUSED)
    print("fused", n, pkg.qap_rlt2_bound(f, 2)["lb"])
    pkg.qap_destroy(f)
torch.cuda.synchronize()
