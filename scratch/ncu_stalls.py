"""Top warp-stall source lines (SASS+CUDA) of an ncu report: python scratch/ncu_stalls.py rep [n]."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
def f(x):
    try: return float(x)
    except ValueError: return 0.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for sec in range(len(hi)):
    h = rows[hi[sec]]
    end = hi[sec + 1] - 1 if sec + 1 < len(hi) else len(rows)
    ia, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    data = [r for r in rows[hi[sec] + 1:end] if len(r) > ia]
    tot = sum(f(r[ia]) for r in data)
    if tot == 0: continue
    print(f"=== file {sec} total {tot:.0f}")
    for r in sorted(data, key=lambda r: -f(r[ia]))[:n]:
        print(f"{f(r[ia]):8.0f} {100*f(r[ia])/tot:5.1f}%  {r[isrc][:110]}")
