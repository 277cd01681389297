"""Shared-memory wavefronts per SASS instruction from an ncu source-page CSV
(tools/diag/ncu_captures.sh output): sass_wavefronts.py NAME [NELT]."""
import collections
import csv
import gzip
import sys

name = sys.argv[1]
nelt = float(sys.argv[2]) if len(sys.argv) > 2 else 196608
rows = list(csv.reader(gzip.open(f"gpurun_out/ncu/{name}_source.csv.gz", "rt")))
h = rows[1]
iS, iW, iWI, iX, iN = (h.index("Source"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"),
                       h.index("Instructions Executed"), h.index("# Samples"))
by = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
top = []
for idx, r in enumerate(rows[2:]):
    if len(r) <= iW:
        continue
    op = r[iS].split()[0] if r[iS].split() else "?"
    if op.startswith("@"):
        op = r[iS].split()[1]
    w, wi, x, ns = (float(r[i] or 0) for i in (iW, iWI, iX, iN))
    k = op.split(".")[0] + ("." + op.split(".")[1] if "." in op and op.startswith(("LDS", "STS", "LDG", "STG")) else "")
    by[k][0] += w; by[k][1] += wi; by[k][2] += x; by[k][3] += ns
    if w:
        top.append((w, wi, x, idx, r[iS].strip()))
print(f"{'op':12s} {'wf/elt':>9s} {'ideal/elt':>9s} {'exec/elt':>9s} {'samples':>8s}")
for k, (w, wi, x, ns) in sorted(by.items(), key=lambda kv: -kv[1][0]):
    if w or x / nelt > 20:
        print(f"{k:12s} {w / nelt:9.1f} {wi / nelt:9.1f} {x / nelt:9.1f} {int(ns):8d}")
print("\ntop shared instructions (wavefronts/elt, ideal, exec/elt, index):")
for w, wi, x, idx, s in sorted(top, reverse=True)[:40]:
    print(f"  {w / nelt:7.2f} {wi / nelt:7.2f} {x / nelt:7.2f} [{idx:5d}] {s}")
