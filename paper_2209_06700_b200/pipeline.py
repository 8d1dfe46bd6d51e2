"""Host-buffer entry point of the stage operator with copy/compute overlap.

`HostStageOperator.apply(u_host, v_host)` computes v = (D_M (x) M + D_K (x) K) u for pinned host
(Q, n) arrays. The x-range is cut into element chunks; chunk c is copied in on an H2D stream, its
K1 window (spk_stage_apply_slab on the full level, elements [c*ce, (c+1)*ce)) runs on the compute
stream once its planes (and the k-plane left halo from chunk c-1) have landed, and its output planes
go back on a D2H stream. PCIe H2D and D2H run concurrently on separate copy engines, so the step
costs about max(H2D, D2H) instead of their sum. The device buffers are double-buffered across calls:
the inputs of call i+1 stream in while the outputs of call i stream out (call i+1's H2D only waits
for the compute that last read its buffer set, two calls back). Every call still ends with the
caller's stream waiting for its D2H, so v_host is complete once that stream is synchronised.
"""

import numpy as np
import torch

from . import _lib
from ._device import ptr


class HostStageOperator:
    def __init__(self, hierarchy, level, DM, DK, chunks=8):
        h = hierarchy
        if h.dim != 3:
            raise ValueError("chunked host pipeline is implemented for 3D levels")
        self.h, self.level = h, level
        self.DM = np.ascontiguousarray(np.asarray(DM, dtype=float))
        self.DK = np.ascontiguousarray(np.asarray(DK, dtype=float))
        self.Q = self.DM.shape[0]
        lvl = h.levels[level]
        self.k, self.E, self.nax = h.degree, lvl.n_elements, lvl.n_per_axis
        self.plane = self.nax * self.nax
        self.n = lvl.n_dofs
        self.chunks = max(1, min(chunks, self.E))
        self.ce = (self.E + self.chunks - 1) // self.chunks
        dev = h.device
        self.us = [torch.empty((self.Q, self.n), dtype=torch.float64, device=dev) for _ in range(2)]
        self.vs = [torch.empty_like(self.us[0]) for _ in range(2)]
        self._parity = 0
        self._cmp_done = [None, None]
        self.s_in = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.current_stream(dev)
        self.launches_per_apply = self.chunks

    def _planes_in(self, c):
        k, ce = self.k, self.ce
        lo = 0 if c == 0 else k * c * ce + 1
        hi = min(k * (c + 1) * ce, self.nax - 1) + 1
        return lo, hi

    def _planes_out(self, c):
        k, ce = self.k, self.ce
        lo = k * c * ce
        hi = min(k * (c + 1) * ce, self.nax - 1)
        if (c + 1) * ce >= self.E:
            hi = self.nax
        return lo, hi

    def apply(self, u_host, v_host):
        Q, P = self.Q, self.plane
        nchunks = (self.E + self.ce - 1) // self.ce
        ev_in = [torch.cuda.Event() for _ in range(nchunks)]
        ev_cmp = [torch.cuda.Event() for _ in range(nchunks)]
        par = self._parity
        self._parity ^= 1
        self.u, self.v = self.us[par], self.vs[par]
        # the caller's prior work on its stream (e.g. filling u_host was host-side; device producers
        # of this call's inputs are not involved) and the compute that last read this buffer set
        if self._cmp_done[par] is not None:
            self.s_in.wait_event(self._cmp_done[par])
        with torch.cuda.stream(self.s_in):
            for c in range(nchunks):
                lo, hi = self._planes_in(c)
                for q in range(Q):  # contiguous per-stage ranges -> plain async DMA
                    self.u[q, lo * P : hi * P].copy_(u_host[q, lo * P : hi * P], non_blocking=True)
                ev_in[c].record(self.s_in)
        for c in range(nchunks):
            self.s_cmp.wait_event(ev_in[c])
            e0, e1 = c * self.ce, min(self.E, (c + 1) * self.ce)
            _lib.call("spk_stage_apply_slab", self.h.ctx, self.level, Q, self.DM.ctypes.data_as(_lib.P_dbl),
                      self.DK.ctypes.data_as(_lib.P_dbl), ptr(self.u), self.n, ptr(self.v), self.n, self.E, e0, e1,
                      1 if e1 == self.E else 0, self.s_cmp.cuda_stream)
            ev_cmp[c].record(self.s_cmp)
        done = torch.cuda.Event()
        done.record(self.s_cmp)
        self._cmp_done[par] = done
        with torch.cuda.stream(self.s_out):
            for c in range(nchunks):
                self.s_out.wait_event(ev_cmp[c])
                lo, hi = self._planes_out(c)
                for q in range(Q):
                    v_host[q, lo * P : hi * P].copy_(self.v[q, lo * P : hi * P], non_blocking=True)
        self.s_cmp.wait_stream(self.s_out)
        return v_host
