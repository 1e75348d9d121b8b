"""Print the repo kernels of an ncu launch-list csv: python scripts/ll.py f.csv [skip_torch]"""
import csv, sys
for f in sys.argv[1:]:
    lines = open(f).read().splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[i:]))
    hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
    print("==", f)
    for r in rows[1:]:
        n = r[ki]
        if 'at::' in n: continue
        print(f"{float(r[vi])/1000:9.1f} us  {n[:60]}")
