"""Warm vs cold B&B: bounded nodes and wall time (batched DFS, one GPU)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1510_02065_b200 as pkg
import qapgen

torch.cuda.set_device(0)
for fam, n in [("nug", 12), ("taib", 13), ("nug", 14), ("nug", 15)]:
    inst = qapgen.make(fam, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D)
    for T in (2, 5, 10):
        for warm in (False, True):
            pkg.qap_bnb_solve(h, T, batch=n, warm=warm) if n <= 13 else None
            t0 = time.perf_counter(); r = pkg.qap_bnb_solve(h, T, batch=n, warm=warm); dt = time.perf_counter() - t0
            print(f"{fam}{n} T={T:2d} {'warm' if warm else 'cold'}: opt={r['opt']} bounded={r['bounded']:6d} "
                  f"pruned={r['pruned']:6d} leaves={r['leaves']:6d} {dt:7.3f}s {r['bounded']/dt:8.0f} nodes/s", flush=True)
    pkg.qap_destroy(h)
