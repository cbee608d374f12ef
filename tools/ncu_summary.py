"""Limiter summary of committed ncu --set full captures (one launch each): throughput fractions of the units that can
bound a kernel, occupancy, issue activity and the top warp-stall reasons. Writes the JSON that bench.py attaches to
each kernel's roofline entry (profiles/ncu_limiters.json).

  python tools/ncu_summary.py WORKLOAD name=REPORT.ncu-rep [name=REPORT ...]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_limiters.json")
KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=subprocess.PIPE,
                         stderr=subprocess.DEVNULL, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    res = {}
    for name, key in KEYS.items():
        if key in h:
            i = h.index(key)
            x = float(v[i].replace(",", ""))
            res[name] = x * SCALE.get(u[i], 1.0) if name.endswith(("bytes", "_us")) else x
    stalls = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    res["top_stalls_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda z: -z[1])[:4]}
    res["report"] = os.path.relpath(rep, ROOT)
    return res


def main():
    workload = sys.argv[1]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data.setdefault(workload, {})
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        data[workload][name] = summary(rep)
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[workload], indent=1))


if __name__ == "__main__":
    main()
