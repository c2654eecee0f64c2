"""Host-side pieces of bench.py (no GPU): the algorithmic byte count the roofline divides by
(16 B per stored D entry, stored entries = n²(n−1)²(n−2)²/2 — P:250-252 halving),
the LAPs per iteration (§8(a) a4 + a5 + a6) and the gating of the committed ncu figures to the
workload they were captured on."""
import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("n", [8, 12, 20, 30, 40])
def test_stored_entries_and_laps(bench, n):
    # brute-force count of stored entries: blocks D{ij,kl} with i < k, j != l, each (n-2)^2
    blocks = sum(1 for i in range(n) for k in range(i + 1, n) for j in range(n) for l in range(n) if j != l)
    assert bench.n_stored(n) == blocks * (n - 2) ** 2
    assert blocks == n * n * (n - 1) * (n - 1) // 2
    # per iteration: one LAP per stored block, n^2 level-1 LAPs, one level-0 LAP
    assert bench.laps_per_iter(n) == blocks + n * n + 1


def test_n30_algorithmic_bytes(bench):
    assert 16 * bench.n_stored(30) == 4_747_276_800


def test_profiled_traffic_only_for_its_workload(bench):
    d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    for k in ("lap2", "transfer"):
        n = int(d[k].get("n", 30))
        assert bench.profiled_traffic(k, n=n) == d[k]["dram_bytes_per_launch"]
        assert bench.profiled_traffic(k, "inst_executed_per_launch", n) == d[k]["inst_executed_per_launch"]
        assert bench.profiled_traffic(k, n=n + 5) is None, "another size moves other bytes"
        assert bench.profiled_traffic(k, n=n, sharded=True) is None, "a shard moves a share"
    assert bench.profiled_traffic("no_such_kernel") is None
