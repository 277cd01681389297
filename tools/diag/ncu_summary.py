"""Per-kernel summary of an `ncu --set full` report (the headline metrics kept
under profiles/). Usage: ncu_summary.py REPORT.ncu-rep "header" > out.txt"""
import csv
import io
import subprocess
import sys

rep, note = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
M = [("gpu__time_duration.sum", "Duration"),
     ("dram__bytes_read.sum", "DRAM read"),
     ("dram__bytes_write.sum", "DRAM write"),
     ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
     ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe active %"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "Issue slots busy %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "Achieved occupancy %"),
     ("launch__registers_per_thread", "Registers/thread"),
     ("launch__shared_mem_per_block_dynamic", "Dynamic smem/block"),
     ("launch__block_size", "Block size"),
     ("launch__grid_size", "Grid size"),
     ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
     ("lts__t_sector_hit_rate.pct", "L2 hit %"),
     ("smsp__inst_executed.sum", "Instructions")]
print(f"# {note}")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print(f"\n## {name.split('(')[0]}")
    for key, label in M:
        if key in hdr:
            i = hdr.index(key)
            print(f"  {label:32s} {r[i]} {units[i]}")
    st = {}
    for i, n in enumerate(hdr):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st[n[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda a: -a[1])[:6]
    print("  stall mix: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))
