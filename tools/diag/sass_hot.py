"""Aggregate an ncu SASS source page (csv, optionally .gz): warp-stall samples
by opcode and the hottest instruction windows. sass_hot.py FILE [window]"""
import csv
import gzip
import io
import sys
from collections import defaultdict

f = sys.argv[1]
txt = gzip.open(f, "rt").read() if f.endswith(".gz") else open(f).read()
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
samp = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(samp(r) for r in data) or 1
by_op = defaultdict(lambda: [0, 0])
stall_cols = [h for h in hdr if h.startswith("stall_")]
by_stall = defaultdict(int)
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    by_op[op][0] += samp(r)
    by_op[op][1] += int(r[ix["Instructions Executed"]] or 0)
    for h in stall_cols:
        by_stall[h] += int(r[ix[h]] or 0)
print(f"total samples {tot}, instructions {sum(v[1] for v in by_op.values())}")
for op, (s, n) in sorted(by_op.items(), key=lambda a: -a[1][0])[:18]:
    print(f"  {op:10s} samples {100 * s / tot:5.1f}%  executed {n}")
st = sum(by_stall.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100 * v / st:.0f}%" for k, v in sorted(by_stall.items(), key=lambda a: -a[1])[:10]))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 40
win = [(sum(samp(r) for r in data[i:i + W]), i) for i in range(0, len(data), W)]
print(f"hottest {W}-instruction windows:")
for s, i in sorted(win, reverse=True)[:8]:
    ops = defaultdict(int)
    for r in data[i:i + W]:
        t = r[ix["Source"]].split()
        o = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")).split(".")[0]
        ops[o] += 1
    print(f"  [{i}..{i + W}) {100 * s / tot:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda a: -a[1])[:6]))
