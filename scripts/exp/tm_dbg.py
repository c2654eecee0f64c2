# debug: wall time (globaltimer, first CTA start to last CTA end) of one level-2 LAP launch and
# the loop cycles of shared-memory vs TMEM warps (ablib/libdbg.so copied over the library)
import ctypes as ct, sys, os
import qapgen, paper_1510_02065_b200 as pkg
n = int(sys.argv[1])
inst = qapgen.taib(n, 1)
h = pkg.qap_rlt2_create(n, inst.F, inst.D)
L = pkg.load_library()
out = (ct.c_ulonglong * 4)()
pkg.qap_rlt2_bound(h, 0)
L.qap_dbg_counts(out)
for it in range(3):
    pkg.qap_rlt2_bound(h, 1)
    L.qap_dbg_counts(out)
    print(f"n={n} TMEM={os.environ.get('QAP_LAP_TMEM','1')} it{it}: lap2 launch {(out[1]-out[0])/1e6:.3f} ms; smem-warp cycles {out[2]:.3e}, TMEM-warp cycles {out[3]:.3e}")
