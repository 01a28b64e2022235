"""DRAM traffic of one GGN product (C3, b=8192) from an ncu --set full capture of its
kernels: sums dram__bytes_read.sum + dram__bytes_write.sum and gpu__time_duration.sum
over the product's launches and writes profiles/<name>.json (read by bench.py)."""
import csv, json, sys
src, out = sys.argv[1], sys.argv[2]
unit = sys.argv[3] if len(sys.argv) > 3 else "one GGN product, C3 784-1024-1024-10, b=8192"
rows = list(csv.reader([l for l in open(src) if l.startswith('"')]))
hdr = rows[0]
units = rows[1] if rows[1] and rows[1][0] == "" else None
data = rows[2:] if units else rows[1:]
col = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    v = r[col[k]].replace(",", "")
    return float(v) if v not in ("", "n/a") else 0.0
kern = []
for r in data:
    kern.append({"kernel": r[col["Kernel Name"]][:80],
                 "us": f(r, "gpu__time_duration.sum") / (1e3 if units and units[col["gpu__time_duration.sum"]] == "ns" else 1.0),
                 "dram_read_B": f(r, "dram__bytes_read.sum"), "dram_write_B": f(r, "dram__bytes_write.sum"),
                 "tensor_pipe_pct": f(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
                 if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in col else None})
tot = sum(k["dram_read_B"] + k["dram_write_B"] for k in kern)
json.dump({"unit_of_work": unit,
           "source": f"ncu --set full --clock-control none (cold-cache replay per kernel), {src}",
           "dram_bytes_per_product": tot, "kernels": kern}, open(out, "w"), indent=1)
print(f"{len(kern)} kernels, DRAM {tot / 1e6:.1f} MB per product")
for k in kern:
    print(f"  {k['us']:7.1f} us rd {k['dram_read_B']/1e6:7.1f} MB wr {k['dram_write_B']/1e6:6.1f} MB tensor {k['tensor_pipe_pct']}  {k['kernel'][:50]}")
