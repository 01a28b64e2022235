"""Summarise an ncu launch-list csv: the kernels of the last GGN product (from the last k_flat_amax)."""
import csv, sys
rows = list(csv.reader([l for l in open(sys.argv[1]) if l.startswith('"')]))
hdr = rows[0]; data = rows[1:]
iN = hdr.index("Kernel Name"); iM = hdr.index("Metric Name"); iV = hdr.index("Metric Value"); iI = hdr.index("ID")
ks = {}
for r in data:
    ks.setdefault(int(r[iI]), {"name": r[iN]})[r[iM]] = r[iV]
ids = sorted(ks)
marker = sys.argv[2] if len(sys.argv) > 2 else "k_flat_amax"
starts = [i for i in ids if marker in ks[i]['name']]
last = [i for i in ids if i >= starts[-1]]
tot = 0
for i in last:
    t = float(ks[i]['gpu__time_duration.sum']) / 1000; tot += t
    rd = float(ks[i].get('dram__bytes_read.sum', 0)) / 1e6; wr = float(ks[i].get('dram__bytes_write.sum', 0)) / 1e6
    print(f"  {t:7.1f} us  rd {rd:6.1f} MB wr {wr:6.1f}  {ks[i]['name'][:60]}")
print("  total", round(tot, 1))
