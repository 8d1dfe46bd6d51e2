"""A/B of libspk variants on the Radau IIA step times (bench.py radau_steps, one GPU session).

usage: python tools/ab_steps.py C1,C3 _variants/a.so _variants/b.so ...
Each variant runs bench.py in its own process (SPK_LIB_PATH); prints ms/step, iterations and the
L2 error per config (the error must not change)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    cfgs = sys.argv[1]
    for lib in sys.argv[2:]:
        path, *sets = lib.split("@")   # variant = path[@ENV=VAL...]
        env = dict(os.environ, SPK_LIB_PATH=os.path.abspath(path), SPK_LIB_LAX="1")
        env.update(dict(kv.split("=", 1) for kv in sets))
        r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu", "--level", "4",
                            "--step-configs", cfgs], cwd=REPO, env=env, capture_output=True, text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if not line:
            print(lib, "FAILED", r.stderr[-1500:])
            continue
        d = json.loads(line[0])
        out = {k: (round(v["ms_per_step"], 3), v["gmres_iterations"][0], v["l2_error"]) for k, v in d["radau_steps"].items()}
        print(os.path.basename(lib), out, flush=True)


if __name__ == "__main__":
    main()
