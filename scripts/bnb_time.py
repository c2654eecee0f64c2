"""Repeatable B&B timing: nug12 seed 1, T=10, batch 12 / 1 / SB; prints min wall time of 5 runs."""
import sys, os, time, inspect
sys.path.insert(0, os.getcwd())
import torch
import paper_1510_02065_b200 as pkg
import qapgen

torch.cuda.set_device(0)
inst = qapgen.nug(12, 1)
h = pkg.qap_rlt2_create(12, inst.F, inst.D, device=0)
sb = "sb_iters" in inspect.signature(pkg.qap_bnb_solve).parameters
for name, kw in (("batch12", dict(batch=12)), ("batch1", dict(batch=1)), ("sb", dict(batch=12, sb_iters=1))):
    if name == "sb" and not sb:
        continue
    pkg.qap_bnb_solve(h, 10, **kw)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = pkg.qap_bnb_solve(h, 10, **kw); ts.append(time.perf_counter() - t0)
    print(name, "min_s=%.4f med_s=%.4f" % (min(ts), sorted(ts)[2]), r)
