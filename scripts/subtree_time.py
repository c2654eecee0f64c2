"""nodes/s: batched DFS (qap_bnb_solve) vs subtree-parallel workers (threads on one GPU)."""
import sys, os, time, threading
sys.path.insert(0, os.getcwd())
import torch
import torch.distributed as dist
import paper_1510_02065_b200 as pkg
from paper_1510_02065_b200 import subtree
import qapgen

torch.cuda.set_device(0)
for fam, n, T in [("nug", 12, 10), ("taib", 13, 10), ("nug", 14, 10)]:
    inst = qapgen.make(fam, n, 1)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D)
    pkg.qap_bnb_solve(h, T, batch=n)
    t0 = time.perf_counter(); r = pkg.qap_bnb_solve(h, T, batch=n); dt = time.perf_counter() - t0
    print(f"{fam}{n} T={T} dfs batch={n}: opt={r['opt']} bounded={r['bounded']} {dt:.3f}s {r['bounded']/dt:.0f} nodes/s", flush=True)
    for W in (1, 2, 4, 8):
        hs = [pkg.qap_rlt2_create(n, inst.F, inst.D, stream=torch.cuda.Stream().cuda_stream) for _ in range(W)]
        for rep in range(2):
            store = dist.HashStore()
            out = [None] * W
            def body(k):
                out[k] = subtree.subtree_bnb(pkg, hs[k], store, k, W, T, target=4 * W, batch=n, sync_every=8, prefix="x/")
            th = [threading.Thread(target=body, args=(k,)) for k in range(W)]
            t0 = time.perf_counter(); [t.start() for t in th]; [t.join() for t in th]; dt = time.perf_counter() - t0
        o = out[0]
        print(f"   W={W}: opt={o['opt']} bounded={o['bounded']} tasks={o['tasks']} donated={o['donated']} {dt:.3f}s {o['bounded']/dt:.0f} nodes/s", flush=True)
        for x in hs: pkg.qap_destroy(x)
    pkg.qap_destroy(h)
