"""Subtree-parallel branch-and-bound across workers.

The paper's multi-GPU search: "The root node of the branch-and-bound tree is performed
by cpu_thread with ID = 0.  Next, at the first Branch, each cpu_thread takes a subtree (or node)
and execute a depth-first search.  When it finished your subtree, the cpu_thread takes another
node that has not been fathomed", with load balancing for unbalanced subtrees.
Here one worker = one GPU (one process per GPU, or threads sharing a GPU in tests):

1. Frontier.  Every worker calls ``qap_bnb_frontier`` with the same arguments: breadth-first
   expansion from the root until a level holds >= ``target`` open nodes.  Bounds are bit-exact
   and deterministic, so every worker gets the same node list without communication (on a
   sharded handle the workers compute each near-root bound together, NCCL).
2. Subtrees.  Workers take node ids from a shared queue and search each subtree depth-first
   with ``qap_bnb_run(root=node)`` on their own single-GPU handle.  Every ``sync_every`` bounded
   nodes and on each improvement a worker publishes its incumbent (atomic min in the store) and
   prunes with the global one.  When workers wait for work, the sync reply asks the busy worker
   to donate: it gives away the unvisited children of its shallowest expanded nodes, which
   become new queue entries (P:307 load balancing).
3. Termination: when every allocated task is done no worker is active, so none can donate
   any more — the queue is final.

The queue is a ``torch.distributed.Store`` (TCPStore across processes, HashStore across
threads): atomic counters ``alloc`` (task ids handed out; the frontier's are 0..F-1),
``taken`` (ids reserved by workers), ``done``; keys ``t/<id>`` (donated nodes), ``ub`` (best
objective) and ``sol/<value>`` (a permutation of that value).  This module is host
scheduling only: every bound runs in the CUDA library through ``qap_bnb_run``.
The optimum is unique; node counts depend on timing (when incumbents arrive) and the
permutation may be any optimal one.
"""
from __future__ import annotations

import json
import math
import time

NONE = 1 << 62  # "no incumbent" in the store's ub key


class SubtreeQueue:
    """Store-backed task queue + incumbent for one search (``prefix`` separates searches)."""

    def __init__(self, store, rank: int, world: int, n_frontier: int, ub0: int = -1, prefix: str = "bnb/"):
        self.s, self.rank, self.world, self.F, self.p = store, rank, world, n_frontier, prefix
        if rank == 0:
            self.s.set(self.p + "ub", str(ub0 if ub0 >= 0 else NONE))
            self.s.add(self.p + "alloc", n_frontier)
            self.s.set(self.p + "ready", "1")
        self.s.wait([self.p + "ready"])
        # start barrier: every worker registered before tasks are taken (donation requests see them)
        self.s.add(self.p + "arrived", 1)
        while self._get("arrived") < world:
            time.sleep(0.0005)

    # -- counters -----------------------------------------------------------------------
    def _get(self, k: str) -> int:
        return self.s.add(self.p + k, 0)

    def global_best(self) -> int:
        v = int(self.s.get(self.p + "ub"))
        return -1 if v >= NONE else v

    def publish(self, best: int, perm) -> int:
        """Atomic min of the incumbent; returns the global best."""
        if best >= 0:
            self.s.set(self.p + f"sol/{best}", json.dumps([int(x) for x in perm]))
            while True:
                cur = self.s.get(self.p + "ub")
                if int(cur) <= best:
                    break
                if self.s.compare_set(self.p + "ub", cur, str(best).encode()) == str(best).encode():
                    break
        return self.global_best()

    def waiting(self) -> int:
        """Workers holding a reserved id that no task has been allocated to yet."""
        return max(0, self._get("taken") - self._get("alloc"))

    def push(self, node: dict) -> None:
        tid = self.s.add(self.p + "alloc", 1) - 1
        self.s.set(self.p + f"t/{tid}", json.dumps(node))

    def take(self, frontier: list, poll: float = 0.001):
        """Next task (its id and node), or None when the search is over."""
        t = self.s.add(self.p + "taken", 1) - 1
        key = self.p + f"t/{t}"
        while True:
            if t < self.F:
                return t, frontier[t]
            if self.s.check([key]):
                return t, json.loads(self.s.get(key))
            d = self._get("done")          # read done before alloc: d == a means that at the
            a = self._get("alloc")         # time done was read no task was active (see module doc)
            if d == a and t >= a:
                return None
            time.sleep(poll)

    def finish(self) -> None:
        self.s.add(self.p + "done", 1)

    def solution(self):
        b = self.global_best()
        return b, (json.loads(self.s.get(self.p + f"sol/{b}")) if b >= 0 else None)

    def gather_stats(self, mine: dict) -> list:
        """All workers' stats dicts (a store barrier)."""
        self.s.set(self.p + f"stats/{self.rank}", json.dumps(mine))
        self.s.wait([self.p + f"stats/{r}" for r in range(self.world)])
        return [json.loads(self.s.get(self.p + f"stats/{r}")) for r in range(self.world)]


def run_worker(q: SubtreeQueue, frontier: list, solve, sync_every: int = 32) -> dict:
    """Take tasks until the queue is final.  solve(node, ub0, sync, donate) -> result dict with
    opt/perm/bounded/leaves/pruned/sb_cut (the signature of qap_bnb_run's hooks)."""
    tot = dict(bounded=0, leaves=0, pruned=0, sb_cut=0, tasks=0, donated=0)
    best, best_perm = -1, None

    def sync(local_best, perm):
        return q.publish(local_best, perm if perm is not None else []), q.waiting()

    def donate(node):
        tot["donated"] += 1
        q.push(node)

    while True:
        got = q.take(frontier)
        if got is None:
            break
        _, node = got
        g = q.global_best()
        r = solve(node, math.inf if g < 0 else float(g), sync, donate)
        for k in ("bounded", "leaves", "pruned", "sb_cut"):
            tot[k] += int(r[k])
        tot["tasks"] += 1
        if r["opt"] >= 0 and (best < 0 or r["opt"] < best):
            best, best_perm = int(r["opt"]), [int(x) for x in r["perm"]]
            q.publish(best, best_perm)
        q.finish()
    tot["opt"] = best
    return tot


def gpu_solver(pkg, h, iters: int, K: float = 0.0, batch: int = 1, sb_iters: int = -1, sync_every: int = 32,
               warm: bool = False):
    """solve() for run_worker on a single-GPU handle h (qap_bnb_run with the hooks)."""
    def solve(node, ub0, sync, donate):
        return pkg.qap_bnb_run(h, iters, K=K, UB0=ub0, batch=batch, sb_iters=sb_iters, root=node, sync=sync,
                               donate=donate, sync_every=sync_every, warm=warm)
    return solve


def subtree_bnb(pkg, h, store, rank: int, world: int, iters: int, target: int | None = None, K: float = 0.0,
                batch: int = 1, sb_iters: int = -1, sync_every: int = 32, prefix: str = "bnb/",
                frontier_handle=None, warm: bool = False) -> dict:
    """Subtree-parallel B&B with one worker per (rank, handle h).  Every worker calls this.
    frontier_handle: handle for phase 1 (e.g. a sharded group handle; default h, each worker
    computing the identical frontier).  warm: warm children below each task's root (the task
    root itself is re-bounded cold on its worker).  Returns the global optimum, a permutation
    of it and the summed counters (frontier counted once)."""
    fh = frontier_handle if frontier_handle is not None else h
    fbatch = batch if getattr(fh, "world", 1) <= 1 else 1
    target = target if target is not None else 4 * world
    nodes, fr = pkg.qap_bnb_frontier(fh, iters, target, K=K, batch=fbatch, sb_iters=sb_iters)
    q = SubtreeQueue(store, rank, world, len(nodes), ub0=fr["opt"], prefix=prefix)
    if fr["opt"] >= 0:
        q.publish(fr["opt"], fr["perm"])
    mine = run_worker(q, nodes, gpu_solver(pkg, h, iters, K, batch, sb_iters, sync_every, warm), sync_every)
    stats = q.gather_stats(mine)
    opt, perm = q.solution()
    out = dict(opt=opt, perm=perm, frontier_nodes=len(nodes), workers=stats)
    for k in ("bounded", "leaves", "pruned", "sb_cut"):
        out[k] = fr[k] + sum(s[k] for s in stats)
    out["tasks"] = sum(s["tasks"] for s in stats)
    out["donated"] = sum(s["donated"] for s in stats)
    return out
