"""Summarise ncu evidence for profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py launches <launches.csv>          # per-kernel shares
    python tools/ncu_summary.py report <report.ncu-rep>          # key counters per kernel
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].strip()
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)  # -> us
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = [{"kernel": k, "launches": cnt[k], "total_ms": round(v / 1e3, 3), "avg_us": round(v / cnt[k], 1),
            "share": round(v / T, 4)} for k, v in tot.most_common()]
    return {"source": path, "total_ms": round(T / 1e3, 3), "kernels": out}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        out.append(d)
    return {"source": path, "kernels": out}


if __name__ == "__main__":
    fn = {"launches": launches, "report": report}[sys.argv[1]]
    print(json.dumps(fn(sys.argv[2]), indent=1))
