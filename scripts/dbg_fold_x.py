import numpy as np, sys
sys.path.insert(0, '.')
import torch; torch.cuda.set_device(0)
import qapgen, oracle, paper_1510_02065_b200 as pkg
n = 17
inst = qapgen.taib(n, 4)
for flags in (0, pkg.QAP_FLAG_BLOCK_LAYOUT):
    hp = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=flags)
    hc = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=flags)
    sp = oracle.State(inst.F, inst.D)
    pkg.qap_rlt2_bound(hp, 2); sp.bound(2)
    I, J = sp.free_maps()
    for a, b in [(0, 0), (16, 3)]:
        pkg.qap_rlt2_fold(hc, hp, int(I[a]), int(J[b]))
        sc = sp.fold(a, b)
        pkg.qap_rlt2_bound(hc, 2); sc.bound(2)
        B, C, D, lb = pkg.qap_rlt2_dual_copy(hc)
        d = np.nonzero(D != sc.D.ravel())[0]
        print("flags", flags, (a, b), "after bound: D diff", len(d), "B", int((B != sc.B.ravel()).sum()), "C", int((C != sc.C.ravel()).sum()), lb, sc.lb)
        if len(d):
            m = 14
            print(d[:10], (d // (m*m))[:10], D[d[:5]], sc.D.ravel()[d[:5]], D.size, sc.D.size)
    pkg.qap_destroy(hp); pkg.qap_destroy(hc)
