"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel name totals and the top launches."""
import csv, sys, collections
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows:
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)  # -> us
    name = r["Kernel Name"][:70]
    agg[name][0] += 1; agg[name][1] += v; tot += v
print(f"total {tot/1e3:.2f} ms over {len(rows)} launches")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"{t/1e3:9.3f} ms {c:6d} {t/c:9.1f} us  {n}")
if len(sys.argv) > 2:
    pat = sys.argv[2]
    sel = [r for r in rows if pat in r["Kernel Name"]]
    for r in sel[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
        print(r["ID"], r["Grid Size"], r["Block Size"], r["Metric Value"], r["Kernel Name"][:40])
