"""A/B of libspk variants on the K1 hot launches (one GPU session; CUDA events, median of 7).

usage: python tools/ab_apply.py _variants/a.so _variants/b.so@SPK_WS=0 ...
Each variant runs in its own process (SPK_LIB_PATH); outputs are compared against the first
variant's (max relative difference), so a faster variant must also be parity-identical."""
import json
import os
import subprocess
import sys

CASES = [  # name, dim, L, k, Q, mode
    ("C2 coupled k4 Q3 (bench)", 3, 6, 4, 3, "coupled"),
    ("C2 coupled constrained", 3, 6, 4, 3, "coupled_c"),
    ("C4 GMRES op k2 Q4 constrained", 3, 7, 2, 4, "coupled_c"),
    ("C4 block STORE k2 x4", 3, 7, 2, 4, "block"),
    ("C5 block STORE k3 x1", 3, 6, 3, 1, "block"),
    ("C5 GMRES op k3 Q3", 3, 6, 3, 3, "coupled_c"),
]

CHILD = r'''
import sys, os, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.tableau import radau_iia
from paper_2209_06700_b200 import measure
out = {}
for name, dim, L, k, Q, mode in json.loads(sys.argv[1]):
    h = build_hierarchy(dim, L, k)
    n = h.levels[L].n_dofs
    g = torch.Generator(device="cuda").manual_seed(1)
    u = torch.rand((Q, n), dtype=torch.float64, device="cuda", generator=g) - 0.5
    v = torch.empty_like(u)
    DM, DK = np.eye(Q), 1e-3 * radau_iia(Q).A
    if mode.startswith("coupled"):
        f = lambda: h.apply_stage_operator(L, DM, DK, u, out=v, constrained=mode.endswith("_c"))
    else:
        lams = [1.5, 2.5, 3.5, 4.5][:Q]
        f = lambda: h.apply_block(L, lams, 1e-3, u, out=v)
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = sorted(measure.event_time(f) for _ in range(7))
    np.save(f"/tmp/ab_{len(out)}_{os.getpid()}.npy", v.cpu().numpy())
    out[name] = (ts[3] * 1e3, f"/tmp/ab_{len(out)}_{os.getpid()}.npy", 16.0 * Q * n / (ts[3] * 1e-3) / 1e9)
print("RESULT" + json.dumps(out))
'''


def main():
    import numpy as np
    libs = sys.argv[1:]
    res = {}
    for lib in libs:
        path, *sets = lib.split("@")   # variant = path[@ENV=VAL[@ENV=VAL...]]
        env = dict(os.environ, SPK_LIB_PATH=os.path.abspath(path), SPK_LIB_LAX="1")
        env.update(dict(kv.split("=", 1) for kv in sets))
        r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(CASES)], env=env, capture_output=True, text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")]
        if not line:
            print(lib, "FAILED", r.stderr[-2000:])
            continue
        res[lib] = json.loads(line[0][6:])
    base = libs[0]
    for name, *_ in CASES:
        row = [name]
        for lib in libs:
            if lib not in res:
                continue
            us, path, gbs = res[lib][name]
            ref = np.load(res[base][name][1])
            d = float(np.abs(np.load(path) - ref).max() / np.abs(ref).max())
            row.append(f"{os.path.basename(lib)}: {us:7.1f} us {gbs:6.0f} GB/s (diff {d:.1e})")
        print(" | ".join(row))


if __name__ == "__main__":
    main()
