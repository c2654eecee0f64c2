"""TMA transfer vs register-load transfer: same bound bits for every n (and fixed nodes)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1510_02065_b200 as pkg
import qapgen
torch.cuda.set_device(0)
ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(range(8, 24))
for N in ns:
    for fixed in ((), ((0, 3),)):
        inst = qapgen.uniform(N, 4)
        out = []
        for fl in (pkg.QAP_FLAG_NO_GRAPH, pkg.QAP_FLAG_NO_GRAPH | pkg.QAP_FLAG_LDG_TRANSFER):
            h = pkg.qap_rlt2_create(N, inst.F, inst.D, flags=fl)
            pkg.qap_rlt2_fix(h, fixed)
            try:
                out.append(pkg.qap_rlt2_bound(h, 2)["lb"])
            except Exception as e:
                out.append(repr(e)[:80])
            pkg.qap_destroy(h)
        print(N, len(fixed), out, out[0] == out[1], flush=True)
