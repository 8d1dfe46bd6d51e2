"""Device plumbing: torch storage, the current CUDA stream, host<->device adaptors.

PyTorch provides device memory and streams only; all arithmetic on the hot path is done by
libspk kernels. Host (numpy) inputs are accepted for drop-in compatibility with callers of the
reference package: they are copied to the device, processed by the same kernels, and copied back.
"""

import numpy as np
import torch


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_06700_b200 needs a CUDA device (sm_100a); no CPU fallback exists")


def stream_ptr(device=None):
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t):
    return t.data_ptr() if t is not None else None


def is_host(x):
    return not isinstance(x, torch.Tensor)


def to_device(x, device, dtype=torch.float64):
    """Return a contiguous fp64 device tensor for x (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        if x.device != device or x.dtype != dtype:
            x = x.to(device=device, dtype=dtype)
        return x.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(device)


def like_input(t, template):
    """Convert the device result t back to the container type of `template`."""
    if is_host(template):
        return t.detach().cpu().numpy()
    return t


class capture_graph:
    """torch.cuda.graph(g) with Python's garbage collector held off for the capture: a collected
    object whose finaliser frees device memory (GridHierarchy -> spk_ctx_destroy -> cudaFree)
    would otherwise invalidate the capture and abort the process."""

    def __init__(self, graph):
        import torch
        self._ctx = torch.cuda.graph(graph)

    def __enter__(self):
        import gc
        self._gc = gc.isenabled()
        gc.collect()
        gc.disable()
        return self._ctx.__enter__()

    def __exit__(self, *exc):
        import gc
        try:
            return self._ctx.__exit__(*exc)
        finally:
            if self._gc:
                gc.enable()
