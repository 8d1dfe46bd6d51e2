"""Dynamic SASS opcode histogram from an ncu source-page CSV (--page source --csv --print-source sass)."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = 1 if "Source" in rows[1] else 0
hdr, data = rows[hi], rows[hi + 1:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iT = hdr.index("Predicated-On Thread Instructions Executed")
ops, thr = collections.Counter(), collections.Counter()
for r in data:
    try:
        n = int(r[iE]); t = int(r[iT])
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[iS])
    if not m:
        continue
    op = m.group(2)
    ops[op] += n
    thr[op] += t
tot = sum(ops.values())
print(f"warp instructions {tot:.3e}")
for o, c in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {o:10s} {c:12d} {100*c/tot:5.1f}%  lanes/instr {thr[o]/max(c,1):5.1f}")
