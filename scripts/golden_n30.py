#!/usr/bin/env python
"""Write tests/golden/n30_nug_seed1.json from the CPU ORACLE only (oracle/, the plain C
implementation of Algorithm 1): the benched configuration (BASELINE.json
config 4: nug30-shaped, seed 1) run for T = 20 dual-ascent iterations.

Stored: LB after iteration 0 (the Gilmore–Lawler bound) and after each iteration (exact
`repr` of the fp64 value), and per first pair (i, j) a BLAKE2b digest of the stored D blocks
D{ij,kl} (i < k; canonical block order, include/qap_rlt2.h export layout) after T = 2, plus
their sum and max, so that a GPU test can compare the whole 2.4 GB tensor without the oracle.
Nothing here comes from the CUDA path.

    python scripts/golden_n30.py            # ~6 min of one core, ~1 min of 8
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import qapgen  # noqa: E402

N, SEED, T, T_D = 30, 1, 20, 2


def group_digests(D, n):
    """Per first pair (i, j): digest, sum and max of its stored blocks (contiguous)."""
    out = []
    t = 0
    for i in range(n):
        for j in range(n):
            cnt = (n - 1 - i) * (n - 1)
            blk = np.ascontiguousarray(D[t:t + cnt])
            t += cnt
            if cnt == 0:
                continue
            out.append({"i": i, "j": j, "blocks": cnt,
                        "blake2b": hashlib.blake2b(blk.tobytes(), digest_size=16).hexdigest(),
                        "sum": repr(float(blk.sum())), "max": repr(float(blk.max()))})
    assert t == D.shape[0]
    return out


def main():
    oracle.build()
    oracle.set_threads(os.cpu_count() or 1)   # bit-identical for every thread count
    inst = qapgen.nug(N, SEED)
    st = oracle.State(inst.F, inst.D)
    t0 = time.time()
    st.iteration0()
    trace = []
    groups = None
    for it in range(1, T + 1):
        st.iteration()
        trace.append(st.lb)
        print(f"iteration {it}: LB = {st.lb!r}  ({time.time() - t0:.0f} s)", flush=True)
        if it == T_D:
            groups = group_digests(st.D, st.n)
    doc = {"cite": "PAPER.md:173-198 (Algorithm 1) with the readings of DESIGN.md §3; BASELINE.json config 4",
           "generator": "scripts/golden_n30.py (calls only oracle/ and qapgen/)",
           "instance": f"qapgen.nug({N}, {SEED})", "N": N, "T": T,
           "lb_glb": repr(st.lb_glb if hasattr(st, "lb_glb") else None),
           "lb_trace": [repr(x) for x in trace],
           "D_after_T": T_D, "D_groups": groups}
    out = oracle.bound(inst.F, inst.D, T=0)
    doc["lb_glb"] = repr(out["lb_glb"])
    path = os.path.join(ROOT, "tests", "golden", f"n{N}_nug_seed{SEED}.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=0)
        f.write("\n")
    print("wrote", path, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
