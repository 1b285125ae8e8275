"""Summarise `ncu --metrics ... --csv` output: one line per (kernel, metric) with the value (sum over launches)."""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    vals = defaultdict(float)
    with open(path) as f:
        rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        try:
            vals[(r[ik].split("(")[0], r[im])] += float(r[iv].replace(",", ""))
        except ValueError:
            pass
    print(path)
    for (k, m), v in sorted(vals.items()):
        print(f"  {k[:60]:60s} {m:75s} {v:.6g}")
