import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1510_02065_b200 as pkg
import qapgen
torch.cuda.set_device(0)
N, fam, fl, dofix, T = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
inst = qapgen.make(fam, N, 1)
h = pkg.qap_rlt2_create(N, inst.F, inst.D, flags=fl)
if dofix:
    pkg.qap_rlt2_fix(h, ())
try:
    print(N, fam, fl, dofix, T, pkg.qap_rlt2_bound(h, T)["lb"])
except Exception as e:
    print(N, fam, fl, dofix, T, "ERR", str(e)[:60])
