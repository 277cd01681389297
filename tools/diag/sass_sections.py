"""Stall-reason mix per SASS index range of an ncu source-page CSV:
sass_sections.py NAME a:b:label [a:b:label ...]"""
import csv
import gzip
import sys

name = sys.argv[1]
rows = list(csv.reader(gzip.open(f"gpurun_out/ncu/{name}_source.csv.gz", "rt")))
h = rows[1]
iN = h.index("# Samples")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iN] or 0) for r in rows[2:] if len(r) > iN)
for spec in sys.argv[2:]:
    a, b, label = spec.split(":")
    seg = rows[2 + int(a):2 + int(b)]
    ns = sum(float(r[iN] or 0) for r in seg)
    mix = {c: sum(float(r[h.index(c)] or 0) for r in seg) for c in reasons}
    top = sorted(mix.items(), key=lambda kv: -kv[1])[:6]
    print(f"{label:10s} {100 * ns / tot:5.1f}%  " + "  ".join(f"{k[6:]} {100 * v / max(ns, 1):.0f}%" for k, v in top))
