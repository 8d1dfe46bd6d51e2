"""Static SASS opcode mix of one kernel in an object file (quick, no GPU): python tools/sass_mix.py obj pattern"""
import collections, re, subprocess, sys
obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if pat not in name:
        continue
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            ops[m.group(2)] += 1
    tot = sum(ops.values())
    print(name[:90], "static instrs", tot)
    print("   ", ", ".join(f"{o}:{c}" for o, c in ops.most_common(20)))
