"""Summarise an ncu source-page CSV (--page source --csv --print-source cuda,sass) by source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = {}; f = None; h = None
for r in rows:
    if r and r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': h = r; ws = h.index('Warp Stall Sampling (All Samples)'); ie = h.index('Instructions Executed'); continue
    if not r or not r[0].isdigit(): continue
    def fl(x):
        try: return float(x)
        except ValueError: return 0.0
    agg[f + ':' + r[0] + ' ' + r[1].strip()[:90]] = (fl(r[ws]), fl(r[ie]))
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f} warp-instructions {toti:.0f}")
print(" stall%  inst%  line")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot:6.1f} {100*v[1]/toti:6.1f}  {k}")
