"""Top stalled SASS instructions of an ncu report's source page (debug aid).
    python tools/stall_top.py report.ncu-rep [N] [reason]"""
import csv, collections, subprocess, sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = collections.Counter()
for r in data:
    for h, i in zip(reasons, ri):
        tot[h[6:]] += f(r[i])
print("total samples %d" % sum(tot.values()), dict(tot.most_common(10)))
key = sys.argv[3] if len(sys.argv) > 3 else None
k = hdr.index("stall_" + key) if key else 2
for j in sorted(range(len(data)), key=lambda j: -f(data[j][k]))[:N]:
    r = data[j]
    top = sorted(((f(r[i]), h[6:]) for h, i in zip(reasons, ri)), reverse=True)[:2]
    print(j, r[0][-5:], int(f(r[2])), top, r[1][:70])
