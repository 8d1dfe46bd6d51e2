"""Build a variant libspk from a git revision's (or the working tree's) csrc into _variants/<name>.so
for A/B timing in one GPU session (SPK_LIB_PATH=_variants/<name>.so):
    python tools/build_variant.py <name> [git-rev]"""
import os, shutil, subprocess, sys, tempfile
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06700_b200 import _build as B
name = sys.argv[1]
rev = sys.argv[2] if len(sys.argv) > 2 else None
extra = os.environ.get("VFLAGS", "").split()
tmp = tempfile.mkdtemp()
src = os.path.join(tmp, "csrc")
if rev:
    os.makedirs(src)
    files = subprocess.run(["git", "ls-tree", "--name-only", rev, "paper_2209_06700_b200/csrc/"],
                           capture_output=True, text=True, check=True).stdout.split()
    for f in files:
        data = subprocess.run(["git", "show", f"{rev}:{f}"], capture_output=True, check=True).stdout
        open(os.path.join(src, os.path.basename(f)), "wb").write(data)
    inc = os.path.join(tmp, "include")
    os.makedirs(inc)
    open(os.path.join(inc, "spk.h"), "wb").write(
        subprocess.run(["git", "show", f"{rev}:include/spk.h"], capture_output=True, check=True).stdout)
    # csrc includes ../../include/spk.h
    os.makedirs(os.path.join(tmp, "a"), exist_ok=True)
    shutil.move(src, os.path.join(tmp, "a", "csrc"))
    src = os.path.join(tmp, "a", "csrc")
    shutil.move(inc, os.path.join(tmp, "include"))
else:
    shutil.copytree(B.CSRC, src)
    inc = os.path.join(tmp, "include")
    os.makedirs(inc, exist_ok=True)
    shutil.copy(os.path.join(B.INCLUDE, "spk.h"), inc)
    os.makedirs(os.path.join(tmp, "a"), exist_ok=True)
    shutil.move(src, os.path.join(tmp, "a", "csrc"))
    src = os.path.join(tmp, "a", "csrc")
def comp(f):
    o = os.path.join(tmp, f.replace(".cu", ".o"))
    r = subprocess.run([B.NVCC, *B.FLAGS, *extra, "-I", os.path.join(tmp, "include"), "-c", os.path.join(src, f), "-o", o],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return o
with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, B.SOURCES))
out = os.path.join(os.path.dirname(B.HERE), "_variants", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", out], check=True)
print(out)
