#!/usr/bin/env python
"""Full branch-and-bound of a synthetic instance on one GPU, in chunks with checkpoints
("checkpoints procedure"), with progress lines: bounded nodes per depth, open nodes, node
rate, and a DFS-progress projection of the total solve time.

    python scripts/bnb_run.py --family taib --n 20 --iters 10 --sb 1 --budget-s 600 --out gpurun_out/x.jsonl

Each chunk is one qap_bnb_run(max_nodes=chunk, resume=...) call; the search state lives in the
checkpoint file between chunks (so a run can also be stopped and resumed later).  Progress
estimate (the standard DFS one): every child subtree of an expanded node counts as an equal
share of its parent's; the explored fraction is the sum, over the expanded nodes on the DFS
stack, of their finished children's shares.
"""
import argparse
import json
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def read_checkpoint(path):
    """Frames (fac, next, nchildren) of the checkpoint written by qap_bnb_run (format v3)."""
    b = open(path, "rb").read()
    pos = [0]

    def get(fmt):
        v = struct.unpack_from("<" + fmt, b, pos[0])
        pos[0] += struct.calcsize("<" + fmt)
        return v[0]

    def getv(fmt):
        n = get("Q")
        sz = struct.calcsize("<" + fmt)
        v = list(struct.unpack_from("<%d%s" % (n, fmt), b, pos[0])) if n else []
        pos[0] += n * sz
        return v

    get("Q"); ver = get("I"); get("Q")
    assert ver == 3, ver
    get("i"); get("i"); get("i"); get("i"); get("d"); get("d")
    get("i"); getv("i"); getv("i")
    get("d"); get("B"); get("q"); getv("i")
    for _ in range(4):
        get("q")
    getv("q")
    nf = get("Q")
    frames = []
    for _ in range(nf):
        fac = getv("i"); getv("i"); fs = getv("i"); getv("i"); getv("d"); getv("d")
        nxt = get("I"); get("B")
        frames.append((len(fac), nxt, len(fs)))
    return frames


def progress(frames):
    frac, share = 0.0, 1.0
    for k, (_, nxt, nch) in enumerate(frames):
        if nch == 0:
            break
        last = k == len(frames) - 1
        done = nxt if last else max(0, nxt - 1)  # the child being searched is the next frame
        frac += share * done / nch
        share /= nch
    return frac


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="taib")
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--sb", type=int, default=1, help="strong branching RLT1 iterations (-1: off)")
    ap.add_argument("--warm", action="store_true")
    ap.add_argument("--batch", type=int, default=0, help="children bounded concurrently (0: N)")
    ap.add_argument("--ub0", type=float, default=float("inf"))
    ap.add_argument("--K", type=float, default=0.0, help="stop a node's ascent when LB'/UB < K (R14)")
    ap.add_argument("--chunk", type=int, default=200)
    ap.add_argument("--budget-s", type=float, default=600)
    ap.add_argument("--ckpt", default=None)
    ap.add_argument("--resume", action="store_true",
                    help="continue the search in --ckpt (time and counters carry over via <ckpt>.json)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch
    import paper_1510_02065_b200 as pkg
    import qapgen
    torch.cuda.set_device(0)
    inst = qapgen.make(a.family, a.n, a.seed)
    h = pkg.qap_rlt2_create(a.n, inst.F, inst.D, device=0)
    ckpt = a.ckpt or f"/tmp/bnb_{a.family}{a.n}_s{a.seed}.ckpt"
    side = ckpt + ".json"
    carried = 0.0
    if a.resume and os.path.exists(ckpt):
        carried = json.load(open(side))["seconds"] if os.path.exists(side) else 0.0
    else:
        a.resume = False
        for f in (ckpt, side):
            if os.path.exists(f):
                os.remove(f)
    out = open(a.out, "a") if a.out else None
    cfg = {"instance": f"{a.family}{a.n}-shaped seed {a.seed}", "N": a.n, "iters_per_node": a.iters,
           "strong_branching": a.sb, "warm_children": a.warm, "batch": a.batch or a.n, "UB0": a.ub0, "K": a.K}

    def emit(d):
        line = json.dumps(d)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()

    emit({"config": cfg, "resumed_from_s": carried if a.resume else None})
    t0 = time.perf_counter() - carried
    t_call = time.perf_counter()
    first, r, last_b, last_t = not a.resume, None, (None if a.resume else 0), t_call
    while True:
        r = pkg.qap_bnb_run(h, a.iters, K=a.K, UB0=a.ub0, batch=a.batch or a.n, sb_iters=a.sb, warm=a.warm,
                            checkpoint_path=ckpt, max_nodes=a.chunk, resume=not first)
        first = False
        torch.cuda.synchronize()
        now = time.perf_counter()
        el = now - t0
        json.dump({"seconds": el}, open(side, "w"))
        prog = 1.0 if r["complete"] else progress(read_checkpoint(ckpt))
        emit({"elapsed_s": el, "bounded": r["bounded"], "leaves": r["leaves"], "pruned": r["pruned"],
              "sb_cut": r["sb_cut"], "open": r["open"], "depth": r["depth_max"], "opt": r["opt"],
              "nodes_per_s_chunk": None if last_b is None else (r["bounded"] - last_b) / max(1e-9, now - last_t),
              "progress": prog, "projected_total_s": el / prog if prog > 0 else None,
              "bounded_by_depth": r["bounded_by_depth"], "complete": r["complete"]})
        last_b, last_t = r["bounded"], now
        if r["complete"] or now - t_call > a.budget_s:
            break
    el = time.perf_counter() - t0
    opt_ok = None
    if r["complete"] and r["opt"] >= 0:
        opt_ok = inst.evaluate([int(x) for x in r["perm"]]) == r["opt"]
    emit({"summary": cfg, "complete": r["complete"], "opt": r["opt"], "perm": [int(x) for x in r["perm"]],
          "perm_evaluates_to_opt": opt_ok, "bounded": r["bounded"], "leaves": r["leaves"], "pruned": r["pruned"],
          "sb_cut": r["sb_cut"], "seconds": el, "nodes_per_s": r["bounded"] / el, "open": r["open"],
          "bounded_by_depth": r["bounded_by_depth"],
          "progress": 1.0 if r["complete"] else progress(read_checkpoint(ckpt)),
          "timer": "host wall clock around the qap_bnb_run chunks (includes checkpoint writes)"})
    pkg.qap_destroy(h)


if __name__ == "__main__":
    main()
