"""SASS of an ncu report's source page in program order with executed counts and stall samples:
    python tools/ncu_loop.py report.ncu-rep [min_exec] [kernel-substring]
(debug aid: read the hot loop of a latency-bound kernel instruction by instruction)"""
import csv
import subprocess
import sys

rep = sys.argv[1]
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
sub = sys.argv[3] if len(sys.argv) > 3 else ""
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
    if sub not in b[0]:
        continue
    print(b[0][:140])
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    isrc = hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[ist] or 0) for r in data)
    print("total samples", tot)
    for j, r in enumerate(data):
        ex = int(r[iex] or 0)
        if ex < min_exec:
            continue
        reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in sc), reverse=True)[:2]
        rs = " ".join(f"{n}:{h}" for n, h in reasons if n)
        print(f"{j:5d} {ex:7d} {int(r[ist] or 0):6d}  {r[isrc].strip()[:72]:72s} {rs}")
