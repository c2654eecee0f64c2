"""The sharded bound across PROCESSES: two processes share the one GPU and
move the transfer's tile exchange and the level-2 all-gather through host-staged
collectives over a gloo process group (qap_host_transport; NCCL refuses two ranks on one
device).  Pack, exchange, apply and all-gather all cross the process boundary; LB trace,
B, C and the assembled D must equal the single-GPU bound bit for bit."""
import os
import socket

import numpy as np
import pytest

import qapgen

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, family, n, T, fixed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1510_02065_b200 as pkg
        from paper_1510_02065_b200.hostcomm import process_group_transport
        inst = qapgen.make(family, n, 3)
        h = pkg.qap_rlt2_create(n, inst.F, inst.D, device=0, world=world, rank=rank,
                                transport=process_group_transport())
        if fixed:
            pkg.qap_rlt2_fix(h, fixed)
        r = pkg.qap_rlt2_bound(h, T, trace=True)
        nB, nC, nD = pkg.qap_rlt2_dual_sizes(h)
        B, C = np.empty(nB), np.empty(nC)
        D = np.full(nD, np.nan)
        lb = __import__("ctypes").c_double()
        pkg._check(pkg.load_library().qap_rlt2_dual_copy(h.ptr, B.ctypes.data, C.ctypes.data, D.ctypes.data,
                                                         __import__("ctypes").byref(lb)), h)
        info = pkg.qap_rlt2_shard_info(h)
        pkg.qap_destroy(h)
        q.put((rank, r["lb_glb"], r["trace"], B, C, D, lb.value, info))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,n,T,fixed", [("nug", 10, 3, ()), ("taib", 12, 2, ((2, 5),)),
                                              ("uniform", 9, 4, ())])
def test_two_processes_equal_single_gpu(family, n, T, fixed):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    import paper_1510_02065_b200 as pkg
    inst = qapgen.make(family, n, 3)
    h = pkg.qap_rlt2_create(n, inst.F, inst.D)
    if fixed:
        pkg.qap_rlt2_fix(h, fixed)
    ref = pkg.qap_rlt2_bound(h, T, trace=True)
    B1, C1, D1, lb1 = pkg.qap_rlt2_dual_copy(h)
    pkg.qap_destroy(h)

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, family, n, T, fixed, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for x in res:
        assert x[1] != "error", x[2]
    D = np.full_like(D1, np.nan)
    owned = 0
    for rank, glb, trace, B, C, Dr, lb, info in res:
        assert glb == ref["lb_glb"]
        assert (trace == ref["trace"]).all()
        assert lb == lb1
        assert (B == B1).all() and (C == C1).all()
        mine = ~np.isnan(Dr)
        assert not (mine & ~np.isnan(D)).any(), "blocks written by both ranks"
        D[mine] = Dr[mine]
        owned += info["blk_hi"] - info["blk_lo"]
    assert owned == n * n * (n - 1) * (n - 1) // 2 or fixed
    assert (D == D1).all()
