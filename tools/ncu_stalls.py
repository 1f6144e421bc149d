"""Aggregate ncu source-page stall samples per kernel and list the top instructions.
python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
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
    print(b[0][:120])
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    isrc = hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = {hdr[i]: sum(int(r[i] or 0) for r in data) for i in sc}
    s = sum(tot.values()) or 1
    print("  samples", sum(int(r[ist] or 0) for r in data), "instructions", sum(int(r[iex] or 0) for r in data))
    print("  ", ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v / s >= 0.02))
    for r in sorted(data, key=lambda r: -int(r[ist] or 0))[:top]:
        reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in sc), reverse=True)[:2]
        print(f"  {r[ist]:>6} {r[iex]:>8}  {r[isrc].strip()[:60]:60s} {reasons}")
