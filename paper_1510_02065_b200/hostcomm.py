"""Host-staged collectives of a sharded bound over torch.distributed.

`process_group_transport(group)` wraps a (gloo or any CPU-capable) process group as the
library's qap_host_transport: the transfer's tile exchange becomes one isend / irecv pair
per peer, the level-2 value all-gather one broadcast per rank.  Plumbing only: the buffers
are the library's staged send / receive slots, moved as they are.  Use it where NCCL cannot
run (several processes sharing one GPU, which NCCL refuses) or to test the sharded data path
across processes without NCCL.
"""
from __future__ import annotations


def process_group_transport(group=None):
    import torch
    import torch.distributed as dist

    from . import host_transport

    def exchange(send, recv, off, count, world, rank):
        reqs = []
        for q in range(world):
            if q == rank or count[q] == 0:
                continue
            a, b = int(off[q]), int(off[q] + count[q])
            reqs.append(dist.isend(torch.from_numpy(send[a:b]), q, group=group))
            reqs.append(dist.irecv(torch.from_numpy(recv[a:b]), q, group=group))
        for r in reqs:
            r.wait()

    def allgather(S, lo, world, rank):
        for q in range(world):
            a, b = int(lo[q]), int(lo[q + 1])
            if b > a:
                dist.broadcast(torch.from_numpy(S[a:b]), q, group=group)

    return host_transport(exchange, allgather)
