"""Top SASS hot spots (warp-stall samples) of an ncu report, with dominant stall reasons.
Usage: python scripts/ncu_hotspots.py <report.ncu-rep> [top_n]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    try:
        n = int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    reasons = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    data.append((n, d["Address"][-5:], d["Source"].strip()[:70], reasons))
tot = sum(x[0] for x in data)
print("total samples", tot)
for n, a, src, rs in sorted(data, reverse=True)[:top]:
    print(f"{n:6d} {100*n/max(tot,1):5.1f}% {a} {src:70s} {' '.join(f'{c}:{v}' for v, c in rs if v)}")
