"""Subtree-parallel B&B scheduler (paper_1510_02065_b200/subtree.py; SURVEY §8(f) NEXT-2;
P:236 workers take subtrees, P:307 load balancing) — host logic on CPU.

The scheduler is driven by a pure-Python DFS worker with the hook semantics of qap_bnb_run
(sync every k nodes / on improvement, donation of the shallowest frames' unvisited
children).  Pins:
  * with pruning disabled every complete permutation is enumerated exactly once across all
    workers (N! leaves-completions), whatever the donations — no subtree lost or duplicated;
  * with pruning (bound = cost of the fixed pairs, valid since costs >= 0) the optimum equals
    brute force;
  * the same over 2 processes (gloo process group + TCPStore on 127.0.0.1).
"""
import itertools
import math
import os
import socket
import threading

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import qapgen
from paper_1510_02065_b200 import subtree


def cost(F, D, perm):
    n = len(perm)
    return int(sum(F[i, k] * D[perm[i], perm[k]] for i in range(n) for k in range(n)))


def brute(F, D):
    n = F.shape[0]
    return min(cost(F, D, p) for p in itertools.permutations(range(n)))


class PyWorker:
    """DFS over one subtree with the hooks of qap_bnb_run (include/qap_rlt2.h)."""

    def __init__(self, F, D, prune=True, sync_every=2):
        self.F, self.D, self.N, self.prune, self.k = F, D, F.shape[0], prune, sync_every
        self.completions = 0

    def bound(self, fac, loc):
        if not self.prune:
            return -math.inf
        return float(sum(self.F[fac[a], fac[b]] * self.D[loc[a], loc[b]]
                         for a in range(len(fac)) for b in range(len(fac))))

    def children(self, fac, loc):
        ffac = [x for x in range(self.N) if x not in fac]
        floc = [x for x in range(self.N) if x not in loc]
        return [(ffac[0], l) for l in floc]

    def solve(self, node, ub0, sync, donate):
        st = dict(bounded=0, leaves=0, pruned=0, sb_cut=0, opt=-1, perm=None)
        UB = ub0
        best = [-1, None]
        improved = [False]

        def cut(lb):
            return lb > UB - 1 + 1e-6

        def leaf(fac, loc):
            st["leaves"] += 1
            ffac = [x for x in range(self.N) if x not in fac]
            floc = [x for x in range(self.N) if x not in loc]
            for p in itertools.permutations(floc):
                perm = [0] * self.N
                for f, l in zip(fac, loc):
                    perm[f] = l
                for f, l in zip(ffac, p):
                    perm[f] = l
                self.completions += 1
                v = cost(self.F, self.D, perm)
                if best[0] < 0 or v < best[0]:
                    best[0], best[1] = v, perm
                    improved[0] = True

        def frame(fac, loc):
            ch = self.children(fac, loc)
            child_leaf = self.N - len(fac) - 1 <= 3
            lbs = [None if child_leaf else self.bound(fac + [f], loc + [l]) for f, l in ch]
            return dict(fac=fac, loc=loc, ch=ch, lb=lbs, next=0, leaf=child_leaf)

        def do_sync():
            nonlocal UB
            g, k = sync(best[0], best[1])
            improved[0] = False
            if best[0] >= 0 and best[0] < UB:
                UB = best[0]
            if g >= 0 and g < UB:
                UB = g
            for Fr in stack:  # donation: shallowest frames first
                if k <= 0:
                    break
                if Fr["leaf"] or Fr["next"] >= len(Fr["ch"]):
                    continue
                for c in range(Fr["next"], len(Fr["ch"])):
                    st["bounded"] += 1
                    if cut(Fr["lb"][c]):
                        st["pruned"] += 1
                        continue
                    f, l = Fr["ch"][c]
                    donate(dict(fac=Fr["fac"] + [f], loc=Fr["loc"] + [l], lb=Fr["lb"][c]))
                    k -= 1
                Fr["next"] = len(Fr["ch"])

        fac, loc = list(node["fac"]), list(node["loc"])
        stack = []
        if self.N - len(fac) <= 3:
            leaf(fac, loc)
        else:
            lb = node.get("lb", math.nan)
            if math.isnan(lb):
                st["bounded"] += 1
                lb = self.bound(fac, loc)
            if cut(lb):
                st["pruned"] += 1
            else:
                stack.append(frame(fac, loc))
        do_sync()
        since = 0
        while stack:
            T = stack[-1]
            if T["next"] >= len(T["ch"]):
                stack.pop()
                continue
            c = T["next"]
            T["next"] += 1
            f, l = T["ch"][c]
            if best[0] >= 0 and best[0] < UB:
                UB = best[0]
            if T["leaf"]:
                leaf(T["fac"] + [f], T["loc"] + [l])
            else:
                st["bounded"] += 1
                since += 1
                if cut(T["lb"][c]):
                    st["pruned"] += 1
                else:
                    stack.append(frame(T["fac"] + [f], T["loc"] + [l]))
            if since >= self.k or improved[0]:
                since = 0
                do_sync()
        do_sync()
        st["opt"], st["perm"] = best[0], best[1]
        return st


def frontier_depth1(N):
    return [dict(fac=[0], loc=[l], lb=-math.inf) for l in range(N)]


def run_threads(F, D, world, prune, frontier, sync_every=2):
    store = dist.HashStore()
    res, workers = [None] * world, []

    def body(r):
        w = PyWorker(F, D, prune, sync_every)
        q = subtree.SubtreeQueue(store, r, world, len(frontier), prefix="t/")
        res[r] = (subtree.run_worker(q, frontier, w.solve), w.completions, q)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(60) for t in th]
    assert all(r is not None for r in res)
    return res


@pytest.mark.parametrize("world", [1, 3])
def test_every_completion_exactly_once(world):
    N = 7
    inst = qapgen.nug(8, 3)
    F, D = inst.F[:N, :N], inst.D[:N, :N]
    res = run_threads(F, D, world, prune=False, frontier=frontier_depth1(N), sync_every=1)
    assert sum(c for _, c, _ in res) == math.factorial(N)
    tasks = sum(r["tasks"] for r, _, _ in res)
    donated = sum(r["donated"] for r, _, _ in res)
    assert tasks == N + donated
    q = res[0][2]
    opt, perm = q.solution()
    assert opt == brute(F, D) and cost(F, D, perm) == opt
    if world > 1:
        assert donated > 0  # idle workers were fed by donation (load balancing)


def test_optimum_with_pruning():
    N = 8
    inst = qapgen.nug(8, 5)
    res = run_threads(inst.F, inst.D, 3, prune=True, frontier=frontier_depth1(N))
    opt, perm = res[0][2].solution()
    assert opt == brute(inst.F, inst.D) and cost(inst.F, inst.D, perm) == opt


def test_single_task_frontier_still_splits():
    """One frontier node, three workers: the others only get work by donation."""
    N = 7
    inst = qapgen.taib(8, 2)
    F, D = inst.F[:N, :N], inst.D[:N, :N]
    res = run_threads(F, D, 3, prune=False, frontier=[dict(fac=[], loc=[], lb=-math.inf)], sync_every=1)
    assert sum(c for _, c, _ in res) == math.factorial(N)
    assert sum(r["donated"] for r, _, _ in res) > 0
    assert sum(1 for r, _, _ in res if r["tasks"] > 0) >= 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc(rank, world, port, sport, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.TCPStore("127.0.0.1", sport, world, rank == 0, wait_for_workers=True)
    N = 7
    inst = qapgen.nug(8, 4)
    F, D = inst.F[:N, :N], inst.D[:N, :N]
    w = PyWorker(F, D, prune=False, sync_every=1)
    q = subtree.SubtreeQueue(store, rank, world, N, prefix="p/")
    r = subtree.run_worker(q, frontier_depth1(N), w.solve)
    stats = q.gather_stats(dict(r, completions=w.completions))
    comp = [None] * world
    dist.all_gather_object(comp, w.completions)  # the gloo path cross-checks the store's view
    opt, perm = q.solution()
    if rank == 0:
        out.put((sum(s["completions"] for s in stats), sum(comp), opt, cost(F, D, perm), brute(F, D)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_gloo():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port, sport = _free_port(), _free_port()
    ps = [ctx.Process(target=_proc, args=(r, 2, port, sport, out)) for r in range(2)]
    [p.start() for p in ps]
    total, total_gloo, opt, c, b = out.get(timeout=120)
    [p.join(60) for p in ps]
    assert all(p.exitcode == 0 for p in ps)
    assert total == total_gloo == math.factorial(7)
    assert opt == c == b
