"""Opcode mix and basic-block weights (instructions, stall samples, top stall reasons) of the first
kernel in an ncu source-page CSV:  ncu -i rep --page source --csv --print-source sass > src.csv;
python tools/ncu_blocks.py src.csv [min_share]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.008
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr) and r[0].startswith("0x"):
        data.append(r)
iA, iS, iE, iW = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
seq = [(int(r[iA], 16), r[iS].strip(), int(r[iE]), int(r[iW]), [int(r[i]) for i in stall_cols]) for r in data]
base = seq[0][0]
tot = sum(x[2] for x in seq); tw = sum(x[3] for x in seq)
print("total warp instrs", tot, "samples", tw)
def opc(s):
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s); return m.group(2) if m else "?"
op = collections.Counter(); st = collections.Counter()
for a, s, e, w, _ in seq:
    op[opc(s)] += e; st[opc(s)] += w
for o, c in op.most_common(25):
    print(f"  {o:10s} {100*c/tot:5.1f}%  stall {100*st[o]/tw:5.1f}%")
blocks = []; cur = []
for x in seq:
    if cur and x[2] != cur[-1][2]:
        blocks.append(cur); cur = []
    cur.append(x)
blocks.append(cur)
for b in blocks:
    w = sum(x[2] for x in b); sw = sum(x[3] for x in b)
    if w / tot < thr and sw / tw < thr:
        continue
    ops = collections.Counter(opc(x[1]) for x in b)
    ss = [sum(x[4][i] for x in b) for i in range(len(stall_cols))]
    top = sorted(zip(ss, [hdr[i][6:] for i in stall_cols]), reverse=True)[:4]
    print(f"{b[0][0]-base:6x}-{b[-1][0]-base:6x} x{b[0][2]:8d} len {len(b):4d} instr {100*w/tot:5.1f}% samples {100*sw/tw:5.1f}%  "
          + ", ".join(f"{o}:{c}" for o, c in ops.most_common(6)) + " | " + ", ".join(f"{n}:{100*v/tw:.1f}" for v, n in top))
