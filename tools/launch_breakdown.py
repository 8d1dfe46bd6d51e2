"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name
(`--grid`: by kernel name and grid size, which separates the multigrid levels)."""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
hdr = rows[0]
iK, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iK].split("(")[0].replace("void <unnamed>::", "").replace("void ", "")
    if "stage_apply_kernel" in r[iK]:
        name = r[iK][r[iK].index("stage_apply_kernel"):].split("(")[0]
    if "--grid" in sys.argv and "Grid Size" in hdr:
        name += "  grid " + r[hdr.index("Grid Size")]
    agg[name][0] += 1
    agg[name][1] += float(r[iV].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: (40 if '--grid' in sys.argv else 1000)]:
    print(f"{100*t/tot:5.1f}%  {t/1e6:8.3f} ms  {n:5d}x  {k[:120]}")
