"""Group the SASS of an ncu source-page CSV into runs of equal execution count (basic blocks) and
print each block's weight and opcode mix: python tools/sass_blocks.py sass.csv [min_share]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = 1 if "Source" in rows[1] else 0
hdr, data = rows[hi], rows[hi + 1:]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
seq = []
for r in data:
    try:
        seq.append((r[iA], r[iS].strip(), int(r[iE])))
    except ValueError:
        pass
tot = sum(n for _, _, n in seq)
blocks, cur = [], []
for a, s, n in seq:
    if cur and n != cur[-1][2]:
        blocks.append(cur)
        cur = []
    cur.append((a, s, n))
blocks.append(cur)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for b in blocks:
    w = sum(x[2] for x in b)
    if w / tot < thr:
        continue
    ops = collections.Counter()
    for _, s, _ in b:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
        if m:
            ops[m.group(2)] += 1
    print(f"{b[0][0][-5:]}-{b[-1][0][-5:]} x{b[0][2]:8d} len {len(b):4d} share {100*w/tot:5.1f}%  " +
          ", ".join(f"{o}:{c}" for o, c in ops.most_common(9)))
