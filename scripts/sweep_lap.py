"""Sweep level-2 LAP launch configurations; report ms per dual-ascent iteration
(CUDA events around bound(T)) and per-kernel averages."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1510_02065_b200 as pkg
import qapgen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
# (flags, lap_cfg)
cfgs = [(0, 0x20), (8, 0x20)] if len(sys.argv) < 3 else [(int(x, 0), 0x20) for x in sys.argv[2].split(",")]
torch.cuda.set_device(0)
inst = qapgen.nug(n, 1)
ref = None
for flags, cfg in cfgs:
    h = pkg.qap_rlt2_create(n, inst.F, inst.D, device=0, flags=flags | pkg.QAP_FLAG_TIME_KERNELS, lap_warps=cfg)
    pkg.qap_rlt2_bound(h, 2)
    pkg.qap_rlt2_kernel_stats(h, reset=True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    r = pkg.qap_rlt2_bound(h, 4)
    s1.record()
    torch.cuda.synchronize()
    st = pkg.qap_rlt2_kernel_stats(h, reset=True)
    ks = {k: round(v["ms"] / max(1, v["launches"]), 4) for k, v in st.items() if v["launches"]}
    ref = r["lb"] if ref is None else ref
    print(f"flags={flags} cfg={hex(cfg)} ms/iter={s0.elapsed_time(s1)/4:.4f} lb_equal={r['lb']==ref} {ks}", flush=True)
    pkg.qap_destroy(h)
