"""Where does a small B&B node's time go?  n = 10 nodes of a nug12 instance, T = 10."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1510_02065_b200 as pkg
import qapgen

torch.cuda.set_device(0)
inst = qapgen.nug(12, 1)
fixes = [((0, a), (1, b)) for a in range(12) for b in range(12) if a != b][:48]
hs = [pkg.qap_rlt2_create(12, inst.F, inst.D, stream=torch.cuda.Stream().cuda_stream) for _ in range(12)]
for h in hs:  # warm graphs
    for fx in fixes[:2]:
        pkg.qap_rlt2_fix(h, fx); pkg.qap_rlt2_bound(h, 10)
torch.cuda.synchronize()
h = hs[0]
t0 = time.perf_counter()
for fx in fixes:
    pkg.qap_rlt2_fix(h, fx); pkg.qap_rlt2_bound(h, 10)
t_seq = (time.perf_counter() - t0) / len(fixes)
# host enqueue cost only
t0 = time.perf_counter()
for k, fx in enumerate(fixes):
    hh = hs[k % 12]
    if k >= 12:
        pkg.qap_rlt2_bound_result(hh)
    pkg.qap_rlt2_fix(hh, fx); pkg.qap_rlt2_bound_async(hh, 10)
t_enq_mixed = (time.perf_counter() - t0) / len(fixes)
for hh in hs:
    pkg.qap_rlt2_bound_result(hh)
torch.cuda.synchronize()
# pure enqueue (no waits) of 12 nodes
t0 = time.perf_counter()
for k in range(12):
    pkg.qap_rlt2_fix(hs[k], fixes[k]); pkg.qap_rlt2_bound_async(hs[k], 10)
t_enq = (time.perf_counter() - t0) / 12
t1 = time.perf_counter()
for k in range(12):
    pkg.qap_rlt2_bound_result(hs[k])
t_wait = (time.perf_counter() - t1)
# GPU time of one node (events)
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
hx = pkg.qap_rlt2_create(12, inst.F, inst.D, stream=s.cuda_stream)
pkg.qap_rlt2_fix(hx, fixes[0]); pkg.qap_rlt2_bound(hx, 10)
with torch.cuda.stream(s):
    e0.record(s)
    for fx in fixes[:10]:
        pkg.qap_rlt2_fix(hx, fx); pkg.qap_rlt2_bound_async(hx, 10)
    e1.record(s)
torch.cuda.synchronize()
print(f"sequential per node {t_seq*1e6:.1f} us; pipelined enqueue+wait per node {t_enq_mixed*1e6:.1f} us; "
      f"pure enqueue per node {t_enq*1e6:.1f} us; wait for 12 {t_wait*1e6:.1f} us; "
      f"GPU time per node (back to back, one stream) {e0.elapsed_time(e1)/10*1e3:.1f} us")
