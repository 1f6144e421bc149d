"""Per-instruction stall samples of one kernel within a SASS offset range
(relative to the function start): python tools/ncu_region.py rep kernel_regex lo hi"""
import csv
import re
import subprocess
import sys

rep, kre, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3], 16), int(sys.argv[4], 16)
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
    ia, ist, isrc = (hdr.index(k) for k in ("Address", "Warp Stall Sampling (All Samples)", "Source"))
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(data[0][ia], 16)
    for r in data:
        off = int(r[ia], 16) - base
        if lo <= off <= hi:
            reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in sc), reverse=True)[:2]
            rs = " ".join(f"{n}:{v}" for v, n in reasons if v)
            print(f"{off:6x} {int(r[ist] or 0):4d} {r[isrc].strip()[:64]:64s} {rs}")
    break
