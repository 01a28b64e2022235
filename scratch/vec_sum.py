"""Summarise an ncu csv of the vector kernels: median time, DRAM bytes, achieved GB/s vs the measured HBM peak."""
import csv, collections, json, statistics as st, sys
rows = list(csv.reader([l for l in open(sys.argv[1]) if l.startswith('"')]))
hdr = rows[0]; data = rows[1:]
iN = hdr.index("Kernel Name"); iM = hdr.index("Metric Name"); iV = hdr.index("Metric Value"); iI = hdr.index("ID")
try:
    peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs") or 6546.6
except Exception:
    peak = 6546.6
ks = {}
for r in data:
    ks.setdefault(int(r[iI]), {"name": r[iN]})[r[iM]] = r[iV].replace(",", "")
agg = collections.defaultdict(list)
for i in sorted(ks):
    k = ks[i]
    agg[k['name'].split('(')[0]].append((float(k['gpu__time_duration.sum']) / 1e3, float(k['dram__bytes_read.sum']) / 1e6,
                                         float(k['dram__bytes_write.sum']) / 1e6))
print(f"{'kernel':26s} {'n':>3s} {'us':>8s} {'rd MB':>8s} {'wr MB':>8s} {'GB/s':>7s} {'% peak':>7s}")
for n, v in agg.items():
    t = st.median(x[0] for x in v); rd = st.median(x[1] for x in v); wr = st.median(x[2] for x in v)
    gbs = (rd + wr) / t * 1e3
    print(f"{n:26s} {len(v):3d} {t:8.1f} {rd:8.1f} {wr:8.1f} {gbs:7.0f} {100 * gbs / peak:6.1f}%")
