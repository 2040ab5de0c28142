"""Summarise an ncu source-page CSV (--page source --csv --print-source cuda,sass):
per source line (stall samples, warp-instructions), top lines, and optional
phase ranges name=file:lo-hi."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
args = sys.argv[2:]
top = int(args[0]) if args and args[0].isdigit() else 40
ranges = [tuple(a.split("=")) for a in args if "=" in a]
agg = {}; f = None
for r in rows:
    if r and r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': h = r; ws = h.index('Warp Stall Sampling (All Samples)'); ie = h.index('Instructions Executed'); continue
    if not r or not r[0].isdigit(): continue
    def fl(x):
        try: return float(x)
        except ValueError: return 0.0
    agg[(f, int(r[0]))] = (fl(r[ws]), fl(r[ie]), r[1].strip()[:100])
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f} warp-instructions {toti:.0f}")
if ranges:
    ph = {}
    for (ff, ln), v in agg.items():
        name = "other"
        for nm, spec in ranges:
            fr, span = spec.split(":"); lo, hi = map(int, span.split("-"))
            if fr == ff and lo <= ln <= hi: name = nm; break
        a = ph.setdefault(name, [0.0, 0.0]); a[0] += v[0]; a[1] += v[1]
    for k, v in sorted(ph.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:12s} stall {100*v[0]/tot:5.1f}%  inst {100*v[1]/toti:5.1f}%  ({v[1]:.3g})")
print(" stall%  inst%  line")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot:6.1f} {100*v[1]/toti:6.1f}  {k[0]}:{k[1]} {v[2]}")
