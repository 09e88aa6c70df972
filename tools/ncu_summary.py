"""Summarise an ncu report (--set full capture) into profiles/: per kernel launch the duration, DRAM
bytes read/written (the roofline `traffic`), DRAM and SM throughput, occupancy and top stall reasons.

  python tools/ncu_summary.py gpurun_out/X/ar_full.ncu-rep profiles/r01/ncu_ar_full.json [label]
Also accepts a launch-list CSV (--metrics gpu__time_duration.sum) and prints per-kernel time shares.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio": "stall_membar",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg_throttle",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio": "stall_drain",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                d[name] = x * SCALE.get(units[i], 1)
        if "dram_read" in d and "dram_write" in d:
            d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
            if d.get("duration"):
                d["dram_GBps"] = d["traffic_bytes"] / d["duration"] / 1e9
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        try:
            tot[r[ki]] = tot.get(r[ki], 0.0) + float(r[vi].replace(",", ""))
        except ValueError:
            pass
    s = sum(tot.values())
    return [{"kernel": k, "total_ns": v, "share": v / s} for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else ""
    data = raw(src) if src.endswith(".ncu-rep") else launches(src)
    with open(dst, "w") as f:
        json.dump({"source": src, "label": label, "rows": data}, f, indent=1)
    for d in data:
        print(json.dumps(d))
