"""One N=30 RLT2 bound (init + iteration 0 + T iterations) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1510_02065_b200 as pkg
import qapgen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lw = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
torch.cuda.set_device(0)
inst = qapgen.nug(n, 1)
h = pkg.qap_rlt2_create(n, inst.F, inst.D, device=0, lap_warps=lw, flags=fl)
print(pkg.qap_rlt2_bound(h, T))
pkg.qap_destroy(h)
