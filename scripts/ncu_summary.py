"""Summarise ncu captures (run here, no GPU): per-kernel DRAM traffic, duration, issue
activity, stall reasons; writes profiles/<round>/ncu_<kernel>.json and updates
profiles/traffic.json (dram bytes per launch, used by bench.py's roofline.traffic)."""
import csv, io, json, subprocess, sys, os

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r); u = next(r); v = next(r)
    return {a: (b, c) for a, b, c in zip(h, u, v)}

def num(x):
    try: return float(x.replace(",", ""))
    except Exception: return None

def summarise(rep, name):
    d = raw(rep)
    g = lambda k: num(d[k][1]) if k in d else None
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = g("dram__bytes_read.sum") * scale[d["dram__bytes_read.sum"][0]]
    wr = g("dram__bytes_write.sum") * scale[d["dram__bytes_write.sum"][0]]
    dur_ms = g("gpu__time_duration.sum") * ({"ms": 1, "us": 1e-3, "ns": 1e-6}[d["gpu__time_duration.sum"][0]])
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): num(v[1])
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    stalls = {k: round(v, 3) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0)) if v and v > 0.05}
    return {"kernel": d.get("Kernel Name", ("", name))[1] if "Kernel Name" in d else name,
            "duration_ms_ncu": dur_ms, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_bytes_per_launch": rd + wr, "dram_GBps": (rd + wr) / dur_ms / 1e6,
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_per_sm": g("sm__warps_active.avg.per_cycle_active"),
            "inst_executed": g("smsp__inst_executed.sum"),
            "registers": g("launch__registers_per_thread"), "stall_reasons_per_issue": stalls,
            "note": "ncu replay (cold caches, serialised, --clock-control none): compare shares, not absolutes"}

if __name__ == "__main__":
    rnd, tag = sys.argv[1], sys.argv[2]
    os.makedirs(f"profiles/{rnd}", exist_ok=True)
    traffic = json.load(open("profiles/traffic.json")) if os.path.exists("profiles/traffic.json") else {}
    for k in ("lap2", "transfer"):
        rep = f"gpurun_out/{tag}_{k}.ncu-rep"
        if not os.path.exists(rep):
            continue
        s = summarise(rep, k)
        json.dump(s, open(f"profiles/{rnd}/ncu_{k}.json", "w"), indent=1)
        traffic[k] = {"n": 30, "dram_bytes_per_launch": s["dram_bytes_per_launch"],
                      "inst_executed_per_launch": s["inst_executed"], "source": f"profiles/{rnd}/ncu_{k}.json",
                      "capture": f"{tag} ncu --set full, N=30 nug seed 1"}
        if k == "lap2":  # warp instructions fall over the ascent: mean over iterations 1..20
            by_it = {}
            for t in (1, 5, 10, 20):
                f = f"gpurun_out/{tag}_lap2_it{t}.csv"
                if os.path.exists(f):
                    for row in csv.reader(open(f)):
                        if len(row) > 3 and row[-3] == "smsp__inst_executed.sum":
                            by_it[t] = float(row[-1].replace(",", ""))
            if len(by_it) == 4:
                ts = sorted(by_it)
                def interp(x):
                    for a, b in zip(ts, ts[1:]):
                        if a <= x <= b:
                            return by_it[a] + (by_it[b] - by_it[a]) * (x - a) / (b - a)
                mean = sum(interp(x) for x in range(1, 21)) / 20
                traffic[k].update({"inst_executed_per_launch": mean, "inst_executed_iteration1": by_it[1],
                                   "inst_executed_by_iteration": {str(t): by_it[t] for t in ts},
                                   "inst_note": "mean over iterations 1..20 interpolated from ncu metric passes at "
                                                f"1, 5, 10, 20 (gpurun_out/{tag}_lap2_it*.csv, copied to profiles/{rnd}/)"})
        print(k, json.dumps(s)[:600])
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
