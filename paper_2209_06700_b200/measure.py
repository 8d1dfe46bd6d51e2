"""Measurement helpers: CUDA-event timing, nvidia-smi clock sampling, peak lookup."""

import json
import os
import subprocess
import threading
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class ClockSampler:
    """Samples SM clocks and throttle reasons with nvidia-smi while active (B200_PROFILING.md)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period_ms=200):
        self.index = index
        self.period = period_ms
        self.proc = None
        self.lines = []
        self._thr = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 f"-i", str(self.index), f"-lms", str(self.period)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._thr = threading.Thread(target=self._read, daemon=True)
            self._thr.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def fp64_peak_tflops(reps=3):
    """DFMA throughput of this GPU, measured now (spk_fp64_probe: 8 independent chains per thread,
    2 x 512-thread CTAs per SM): the denominator of the bench line's fp64_pipe fraction."""
    from . import _lib
    from ._device import stream_ptr

    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    ctas, threads, iters = 2 * sms, 512, 4096
    sink = torch.empty(1024, dtype=torch.float64, device="cuda")
    st = stream_ptr(sink.device)
    run = lambda: _lib.call("spk_fp64_probe", ctas, threads, iters, sink.data_ptr(), st)
    run()
    best = min(event_time(run) for _ in range(reps))
    flops = 2.0 * 8 * 16 * iters * ctas * threads
    return flops / (best * 1e-3) / 1e12


def event_time(fn, stream=None):
    """Run fn() between two CUDA events on the current stream; returns milliseconds."""
    s = stream or torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1)
