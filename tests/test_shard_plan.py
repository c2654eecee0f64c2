"""Host logic of the multi-GPU sharding, no GPU: the facility partition,
the per-rank tile lists and the symmetric exchange-slot layout; plus a world_size-2 gloo
run that exchanges slot-addressed payloads the way the NCCL all-to-all does."""
import os
import socket

import numpy as np
import pytest


@pytest.fixture(scope="module")
def pkg():
    from paper_1510_02065_b200 import build
    build.build()
    import paper_1510_02065_b200 as p
    p.load_library()
    return p


def nblk(n):
    return n * n * (n - 1) * (n - 1) // 2


def triples(n):
    return [(i, k, p) for i in range(n) for k in range(i + 1, n) for p in range(k + 1, n)]


def owners(pkg, n, G):
    """Facility owner from the rank-major block ranges and the tile lists."""
    plans = [pkg.qap_shard_plan(n, G, r) for r in range(G)]
    return plans


@pytest.mark.parametrize("n", [5, 8, 12, 30])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_plan_partition_and_tiles(pkg, n, G):
    plans = [pkg.qap_shard_plan(n, G, r) for r in range(G)]
    blk = plans[0]["blk_lo"]
    for p in plans:
        assert (p["blk_lo"] == blk).all(), "every rank computes the same partition"
    assert blk[0] == 0 and blk[-1] == nblk(n) and (np.diff(blk) >= 0).all()
    loads = np.diff(blk)
    if n >= 12:  # LPT: within 15% of the mean, or the largest facility (granularity)
        assert loads.max() <= max(1.15 * loads.mean(), n * (n - 1) * (n - 1)) + n * n, "LPT balance"
    nt = -(-n // 8)
    nt3 = nt ** 3
    tri = triples(n)
    # every tile appears on the owner of its facility i and of its facility k
    seen = {}
    for r, p in enumerate(plans):
        # the local tiles first (transferred during the exchange), then the shared ones by
        # exchange piece c: slot s of the S slots shared with peer q (range starting at off_q)
        # lies in piece c when floor(c S / 4) <= s - off_q < floor((c + 1) S / 4); ascending
        # global tile id within each group
        loc = p["kind"] == 0
        nl = int(loc.sum())
        assert loc[:nl].all() and not loc[nl:].any(), "local tiles first"
        assert (np.diff(p["tiles"][:nl]) > 0).all(), "local tiles ascending"
        off = np.concatenate([[0], np.cumsum(p["peer_slots"])])
        pieces = []
        for s in p["slot"][nl:]:
            q = int(np.searchsorted(off, s, side="right") - 1)
            S, rel = int(p["peer_slots"][q]), int(s - off[q])
            pieces.append(max(c for c in range(4) if S * c // 4 <= rel))
        pieces = np.array(pieces, np.int64)
        assert (np.diff(pieces) >= 0).all(), "shared tiles ordered by exchange piece"
        for c in range(4):
            t = p["tiles"][nl:][pieces == c]
            assert (np.diff(t) > 0).all(), "ascending within a piece"
        for t, kind in zip(p["tiles"], p["kind"]):
            seen.setdefault(int(t), []).append((r, int(kind)))
    assert len(seen) == len(tri) * nt3
    fac_owner = {}
    for t, lst in seen.items():
        i, k, _ = tri[t // nt3]
        kinds = sorted(kd for _, kd in lst)
        if kinds == [0]:
            (r, _), = lst
            for f in (i, k):
                assert fac_owner.setdefault(f, r) == r
        else:
            assert kinds == [1, 2]
            agg = [r for r, kd in lst if kd == 1][0]
            hold = [r for r, kd in lst if kd == 2][0]
            assert agg != hold
            assert fac_owner.setdefault(i, agg) == agg
            assert fac_owner.setdefault(k, hold) == hold


@pytest.mark.parametrize("n,G", [(8, 2), (12, 3), (30, 8)])
def test_slot_layout_symmetric(pkg, n, G):
    """For every peer pair (r, s) the shared tiles, sorted by global id, occupy the same
    positions in r's slot range for s and in s's slot range for r."""
    plans = [pkg.qap_shard_plan(n, G, r) for r in range(G)]
    offs = [np.concatenate([[0], np.cumsum(p["peer_slots"])]) for p in plans]
    lists = {}
    for r, p in enumerate(plans):
        for t, kind, slot in zip(p["tiles"], p["kind"], p["slot"]):
            if kind == 0:
                continue
            s = int(np.searchsorted(offs[r], slot, side="right") - 1)
            lists.setdefault((r, s), []).append((int(slot - offs[r][s]), int(t)))
    for (r, s), lst in lists.items():
        other = lists[(s, r)]
        assert sorted(lst) == sorted(other)
        assert [t for _, t in sorted(lst)] == sorted(t for _, t in lst)
        assert plans[r]["peer_slots"][s] == plans[s]["peer_slots"][r] == len(lst)


def _gloo_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1510_02065_b200 as pkg
        p = pkg.qap_shard_plan(n, world, rank)
        kSlot = 512
        send = torch.full((int(p["peer_slots"].sum()) * kSlot,), -1.0, dtype=torch.float64)
        # payload of each shared tile: its global tile id (what the partner must find there)
        for t, kind, slot in zip(p["tiles"], p["kind"], p["slot"]):
            if kind:
                send[slot * kSlot:(slot + 1) * kSlot] = float(t)
        recv = torch.empty_like(send)
        sizes = [int(x) * kSlot for x in p["peer_slots"]]
        dist.all_to_all_single(recv, send, output_split_sizes=sizes, input_split_sizes=sizes)
        ok = True
        for t, kind, slot in zip(p["tiles"], p["kind"], p["slot"]):
            if kind:
                ok &= bool((recv[slot * kSlot:(slot + 1) * kSlot] == float(t)).all())
        q.put((rank, ok, int(p["peer_slots"].sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [6, 12])
def test_gloo_world2_exchange_layout(pkg, n):
    import torch.multiprocessing as mp
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert res[0][2] == res[1][2] > 0


def _hostcomm_worker(rank, world, port, n, q):
    """The host-staged transport's callbacks (paper_1510_02065_b200/hostcomm.py) over gloo,
    driven exactly as the library drives them: staged slot buffers with the plan's per-peer
    offsets / counts, then the rank-major all-gather of level-2 values."""
    import ctypes as ct

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1510_02065_b200 as pkg
        from paper_1510_02065_b200.hostcomm import process_group_transport
        t = process_group_transport()
        p = pkg.qap_shard_plan(n, world, rank)
        kSlot = 512
        slots = p["peer_slots"].astype(np.int64)
        off = np.concatenate([[0], np.cumsum(slots)[:-1]]).astype(np.int64) * kSlot
        cnt = slots * kSlot
        cnt[rank] = 0
        send = np.full(int(slots.sum()) * kSlot + 1, -1.0)
        for tid, kind, slot in zip(p["tiles"], p["kind"], p["slot"]):
            if kind:
                send[slot * kSlot:(slot + 1) * kSlot] = float(tid)
        recv = np.zeros_like(send)
        dp = ct.POINTER(ct.c_double)
        ip = ct.POINTER(ct.c_int64)
        rc = t.exchange(None, send.ctypes.data_as(dp), recv.ctypes.data_as(dp), off.ctypes.data_as(ip),
                        cnt.ctypes.data_as(ip), world, rank)
        ok = rc == 0
        for tid, kind, slot in zip(p["tiles"], p["kind"], p["slot"]):
            if kind:
                ok &= bool((recv[slot * kSlot:(slot + 1) * kSlot] == float(tid)).all())
        lo = p["blk_lo"].astype(np.int64)
        S = np.full(int(lo[-1]), -1.0)
        S[lo[rank]:lo[rank + 1]] = np.arange(lo[rank], lo[rank + 1], dtype=np.float64)
        rc = t.allgather(None, S.ctypes.data_as(dp), lo.ctypes.data_as(ip), world, rank)
        ok &= rc == 0 and bool((S == np.arange(lo[-1], dtype=np.float64)).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 12])
def test_gloo_world2_host_transport(pkg, n):
    """world_size 2 on CPU: the host transport's exchange delivers every shared tile's slots
    to its partner and the all-gather leaves every rank with all level-2 values."""
    import torch.multiprocessing as mp
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hostcomm_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok in res), res
