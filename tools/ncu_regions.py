"""Attribute SASS stall samples and instruction counts to regions delimited by BAR.SYNC."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {r: hdr.index(r) for r in reasons}
region = 0
agg = collections.defaultdict(lambda: collections.Counter())
ops = collections.defaultdict(lambda: collections.Counter())
for r in data:
    src = r[iS]
    if "BAR.SYNC" in src:
        region += 1
    for rs in reasons:
        v = r[idx[rs]]
        if v.isdigit(): agg[region][rs] += int(v)
    e = r[iE]
    if e.isdigit():
        t = src.split(); o = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
        ops[region][o] += int(e)
for reg in sorted(agg):
    tot = sum(agg[reg].values())
    if tot < 50: continue
    top = ", ".join(f"{k[6:]}:{v}" for k, v in agg[reg].most_common(6))
    ins = sum(ops[reg].values())
    print(f"region {reg}: samples {tot}  instr {ins}  DFMA {ops[reg]['DFMA']}  | {top}")
