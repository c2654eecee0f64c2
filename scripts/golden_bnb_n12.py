#!/usr/bin/env python
"""Write tests/golden/n12_nug_seed1_bnb.json (BASELINE.json config 2: nug12-shaped, seed 1,
full branch-and-bound) from the CPU ORACLE only:

* the brute-force optimum over all 12! permutations (oracle_qap_bruteforce: the objective of
  PAPER.md:84 enumerated; independent of the bound) and the first optimal permutation;
* the oracle B&B (oracle_bnb; reading R18-R22) with T = 10 RLT2
  iterations per node: cold children, strong branching (RLT1, 1 iteration) and warm
  children (reading R31) — optimum, permutation, bounded nodes, leaves, pruned, RLT1 cuts.

    python scripts/golden_bnb_n12.py        # ~2 min of one core
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import qapgen  # noqa: E402

N, SEED, T = 12, 1, 10


def main():
    oracle.build()
    inst = qapgen.nug(N, SEED)
    t0 = time.time()
    opt, perm = oracle.qap_bruteforce(inst.F, inst.D)
    print(f"brute force: {opt} {list(perm)} ({time.time() - t0:.0f} s)", flush=True)
    doc = {"cite": "BASELINE.json config 2; PAPER.md:84 (objective), P:236-238 and P:305 (B&B, node counts), "
                   "P:254 (strong branching); DESIGN.md readings R15, R18-R22, R31",
           "generator": "scripts/golden_bnb_n12.py (calls only oracle/ and qapgen/)",
           "instance": f"qapgen.nug({N}, {SEED})", "N": N, "T": T,
           "bruteforce": {"opt": int(opt), "first_perm": [int(x) for x in perm]}, "bnb": {}}
    for name, kw in (("cold", {}), ("strong_branching", {"sb_iters": 1}), ("warm", {"warm": True})):
        t1 = time.time()
        o = oracle.bnb(inst.F, inst.D, T=T, **kw)
        doc["bnb"][name] = {"kwargs": kw, "opt": int(o["opt"]), "perm": [int(x) for x in o["perm"]],
                            "bounded": int(o["bounded"]), "leaves": int(o["leaves"]), "pruned": int(o["pruned"]),
                            "sb_cut": int(o["sb_cut"])}
        print(name, doc["bnb"][name], f"({time.time() - t1:.0f} s)", flush=True)
    path = os.path.join(ROOT, "tests", "golden", f"n{N}_nug_seed{SEED}_bnb.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
