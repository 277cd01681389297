"""Convert an `ncu --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` log into the launch list kept under profiles/
(id,kernel,time_ns,dram_read_bytes,dram_write_bytes).
Usage: ncu_to_launches.py NCU_CSV OUT_CSV "header comment" """
import csv
import sys

src, out, note = sys.argv[1], sys.argv[2], sys.argv[3]
rows = {}
order = []
scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
lines = [ln for ln in open(src) if ln.startswith('"')]
for r in csv.DictReader(lines):
    key = r["ID"]
    if key not in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").strip().replace(",", ";")
        rows[key] = {"kernel": name}
        order.append(key)
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    rows[key][r["Metric Name"]] = v
with open(out, "w") as fh:
    fh.write(f"# {note}\n# cold-cache, serialised per-launch times: compare SHARES, not absolutes\n")
    fh.write("id,kernel,time_ns,dram_read_bytes,dram_write_bytes\n")
    for i, k in enumerate(order):
        r = rows[k]
        fh.write(f"{i},{r['kernel']},{r.get('gpu__time_duration.sum', 0):.0f},"
                 f"{r.get('dram__bytes_read.sum', 0):.0f},{r.get('dram__bytes_write.sum', 0):.0f}\n")
