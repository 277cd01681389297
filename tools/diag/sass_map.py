"""Windowed map of an ncu source-page CSV: samples, executions and dominant
opcodes per window of W SASS instructions: sass_map.py NAME [W] [NELT]."""
import collections
import csv
import gzip
import sys

name = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 100
nelt = float(sys.argv[3]) if len(sys.argv) > 3 else 196608
rows = list(csv.reader(gzip.open(f"gpurun_out/ncu/{name}_source.csv.gz", "rt")))
h = rows[1]
iS, iN, iX = h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
body = [r for r in rows[2:] if len(r) > iX]
tot = sum(float(r[iN] or 0) for r in body)
for a in range(0, len(body), W):
    seg = body[a:a + W]
    ns = sum(float(r[iN] or 0) for r in seg)
    if ns / tot < 0.003:
        continue
    ops = collections.Counter((r[iS].split()[1] if r[iS].strip().startswith("@") else r[iS].split()[0]).split(".")[0]
                              for r in seg if r[iS].strip())
    ex = max(float(r[iX] or 0) for r in seg) / nelt
    mix = {c: sum(float(r[h.index(c)] or 0) for r in seg) for c in reasons}
    top = sorted(mix.items(), key=lambda kv: -kv[1])[:3]
    print(f"{a:5d} {100 * ns / tot:5.1f}% x{ex:4.1f} " + " ".join(f"{k}:{v}" for k, v in ops.most_common(4)) +
          " | " + " ".join(f"{k[6:]} {100 * v / max(ns, 1):.0f}%" for k, v in top))
