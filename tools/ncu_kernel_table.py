"""Summarise ncu --set full reports (one launch each) into the profiles/ kernel table:
python tools/ncu_kernel_table.py out.txt "title::report.ncu-rep" ..."""
import csv, io, subprocess, sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
out = open(sys.argv[1], "w")
out.write("# ncu --set full --clock-control none, one launch per kernel (one B200); tools/ncu_kernels.sh\n"
          "# DRAM GB/s = (read + write) / duration. HBM-bound kernels are judged against 6546.6 GB/s (MEASURED_PEAKS);\n"
          "# K1 launches by the FP64 pipe (34.2 TF/s measured DFMA peak) -- see DESIGN.md §3\n")
for arg in sys.argv[2:]:
    title, rep = arg.rsplit("::", 1)
    res = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(res)))
    if len(rows) < 3:
        out.write(f"\n## {title}: no data\n")
        continue
    h, u, d = rows[0], rows[1], dict(zip(rows[0], rows[2]))
    out.write(f"\n## {title}\n")
    for k in KEYS:
        if k in d:
            out.write(f"  {k:66s} {d[k]} {u[h.index(k)]}\n")
    try:
        unit = lambda k: SCALE.get(u[h.index(k)], 1.0)
        t = float(d["gpu__time_duration.sum"]) * unit("gpu__time_duration.sum")
        by = float(d["dram__bytes_read.sum"]) * unit("dram__bytes_read.sum") + \
             float(d["dram__bytes_write.sum"]) * unit("dram__bytes_write.sum")
        out.write(f"  => DRAM {by / t / 1e9:.0f} GB/s over {t * 1e6:.1f} us\n")
    except (KeyError, ValueError):
        pass
