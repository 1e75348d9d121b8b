"""Summarise ncu launch-list csv files: per kernel mean us of the last iteration(s)."""
import csv, sys, collections
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]; n, v = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(r[n], float(r[v].replace(",", ""))) for r in rows[hi + 1:] if "moe::" in r[n]]
    agg = collections.OrderedDict()
    for name, t in ks:
        agg.setdefault(name.split("(")[0][-40:], []).append(t / 1e3)
    print(f, " | ".join(f"{k.replace('void moe::','')}: {sum(x)/len(x):.1f}" for k, x in agg.items()))
