"""Group an ncu source-page CSV of beam_fast_kernel by source-line ranges
(phases of a beam stage): stall samples and executed warp-instructions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ranges = [tuple(x.split("=")) for x in sys.argv[2:]]  # name=file:lo-hi
agg = {}; f = None; tot_s = tot_i = 0.0
for r in rows:
    if r and r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': h = r; ws = h.index('Warp Stall Sampling (All Samples)'); ie = h.index('Instructions Executed'); continue
    if not r or not r[0].isdigit(): continue
    try: sv, iv = float(r[ws] or 0), float(r[ie] or 0)
    except ValueError: continue
    tot_s += sv; tot_i += iv
    ln = int(r[0]); name = "other"
    for nm, spec in ranges:
        ff, span = spec.split(":"); lo, hi = map(int, span.split("-"))
        if ff == f and lo <= ln <= hi: name = nm; break
    a = agg.setdefault(name, [0.0, 0.0]); a[0] += sv; a[1] += iv
print(f"samples {tot_s:.0f} warp-instructions {tot_i:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:12s} stall {100*v[0]/tot_s:5.1f}%  inst {100*v[1]/tot_i:5.1f}%  ({v[1]:.3g})")
