"""Summarise an ncu report: headline metrics, stall mix, and the hottest source
lines (warp-stall samples). Usage: ncu_lines.py REPORT.ncu-rep [N] [kernel-regex]."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16
filt = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + filt, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:75s} {v[i]} {units[i]}")
tot = {}
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        try:
            tot[n[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
        except ValueError:
            pass
s = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{k} {x / s * 100:.1f}%" for k, x in sorted(tot.items(), key=lambda a: -a[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + filt,
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
hdr = f = None
for row in csv.reader(io.StringIO(src)):
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 8:
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    a = agg[(f, ln)]
    for j, col in ((0, 4), (1, 7)):
        try:
            a[j] += float(row[col] or 0)
        except ValueError:
            pass
    for j, n in enumerate(hdr):
        if n.startswith("stall_") and "(" not in n:
            try:
                a[2][n] += float(row[j] or 0)
            except ValueError:
                pass
tot = sum(a[0] for a in agg.values()) or 1
for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    top = ", ".join(f"{n[6:]}:{x / a[0] * 100:.0f}" for n, x in a[2].most_common(3)) if a[0] else ""
    print(f"{k[0]:26s}{k[1]:5d} {a[0] / tot * 100:5.1f}%  inst {a[1]:.3g}  {top}")
