"""Sum ncu stall samples of one kernel over SASS offset ranges (relative to
the function start) and list per-reason totals.
python tools/ncu_ranges.py report.ncu-rep kernel_regex start:end [start:end ...]"""
import csv
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
ranges = [tuple(int(x, 16) for x in r.split(":")) for r in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.split("\n")
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = [line]
        blocks.append(cur)
    elif cur is not None:
        cur.append(line)
for b in blocks:
    if not re.search(kre, b[0]):
        continue
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    ia, ist, isrc, iex = (hdr.index(k) for k in ("Address", "Warp Stall Sampling (All Samples)", "Source",
                                                 "Instructions Executed"))
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(data[0][ia], 16)
    tot_all = sum(int(r[ist] or 0) for r in data)
    print(b[0][:110], "samples", tot_all)
    for lo, hi in ranges:
        sel = [r for r in data if lo <= int(r[ia], 16) - base <= hi]
        s = sum(int(r[ist] or 0) for r in sel)
        ex = [int(r[iex] or 0) for r in sel]
        reasons = {hdr[i][6:]: sum(int(r[i] or 0) for r in sel) for i in sc}
        rs = ", ".join(f"{k} {v}" for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:6] if v)
        print(f"  [{lo:#x},{hi:#x}] {len(sel)} instr, max exec {max(ex) if ex else 0}, samples {s}: {rs}")
        if len(sys.argv) > 1 and "-v" in sys.argv[0:1]:
            pass
    break
