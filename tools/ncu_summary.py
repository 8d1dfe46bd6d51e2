"""Summarise an ncu report: key raw metrics, stall breakdown, opcode mix (top), hottest SASS."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr, units = raw[0], raw[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]
for row in raw[2:]:
    d = dict(zip(hdr, row))
    for k in keys:
        if k in d: print(f"{k:70s} {d[k]} {units[hdr.index(k)]}")
    print("stalls (warps per issue):")
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                if float(v) > 0.05: print(f"   {h[34:-23]:30s} {float(v):.2f}")
            except ValueError: pass
if "--sass" in sys.argv:
    rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
    h = rows[1]; data = rows[2:]
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    op, st = collections.Counter(), collections.Counter()
    for r in data:
        try: e, w = int(r[iE]), int(r[iW])
        except ValueError: continue
        t = r[iS].split(); o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        op[o] += e; st[o] += w
    tot = sum(op.values()); tw = sum(st.values())
    print("total warp instructions", tot)
    for o, c in op.most_common(16): print(f"   {o:10s} {100*c/tot:5.1f}%  stall {100*st[o]/tw:5.1f}%")
