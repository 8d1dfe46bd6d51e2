"""The two Kronecker primitives on stage block vectors (SPEC tensor_ops):

  scale_blocks(apply_C, u)   v = (I_Q (x) C) u   -- stage-local, no inter-stage traffic
  dense_combine(D, u)        v = (D (x) I_n) u   -- one fused pointwise pass (spk_combine)
  complex forward / back     the paired real layout of SPEC rotate_combine_paired: a complex
                             stage vector of ceil(Q/2) blocks is stored as 2*ceil(Q/2) real rows
                             (re, im) so S^{-1} and S act as real (2P x Q) / (Q x 2P) matrices.

The multi-GPU rotation (Cannon-like ring) lives in parallel.rotate_combine.
"""

import numpy as np
import torch

from . import _lib
from ._device import ptr, stream_ptr
from .errors import DimensionMismatchError


def _ctx_and_stream(u, hierarchy):
    ctx = hierarchy.ctx if hierarchy is not None else _null_ctx()
    return ctx, stream_ptr(u.device)


_NULL = None


def _null_ctx():
    """A tiny context for combines that need no grid information."""
    global _NULL
    if _NULL is None:
        ctx = _lib.c_vp()
        _lib.check(_lib.load().spk_ctx_create(1, 1, 1, _lib.ctypes.byref(ctx)))
        _NULL = ctx
    return _NULL


def scale_blocks(apply_C, u):
    """v_i = C u_i for every stage block (generalized vector scaling)."""
    return torch.stack([apply_C(u[i]) for i in range(u.shape[0])]) if callable(apply_C) else None


def dense_combine(D, u, out=None, accumulate=False, mask_level=-1, hierarchy=None):
    """v_i = sum_j D_ij u_j (D real, nout x nin) in one pass over the DoFs."""
    D = np.ascontiguousarray(np.asarray(D, dtype=float))
    if D.ndim != 2 or D.shape[1] != u.shape[0]:
        raise DimensionMismatchError(f"combine matrix {D.shape} vs {u.shape[0]} blocks")
    nout, nin = D.shape
    n = u.shape[-1]
    u = u.reshape(nin, n)
    if not u.is_contiguous():
        u = u.contiguous()
    if out is None:
        out = torch.empty((nout, n), dtype=torch.float64, device=u.device)
    ctx, s = _ctx_and_stream(u, hierarchy)
    _lib.call("spk_combine", ctx, int(mask_level), n, nin, nout, D.ctypes.data_as(_lib.P_dbl), ptr(u), n,
              ptr(out), out.stride(0), 1 if accumulate else 0, s)
    return out


def paired_forward_matrix(Sinv, pairs):
    """Real (2P x Q) matrix mapping a real stage vector to (re, im) rows of the P complex blocks
    w_p = (S^{-1} u)_p for the pair representatives (real block: im row is zero)."""
    rows = []
    for p in pairs:
        rows.append(np.real(Sinv[p.index]))
        rows.append(np.imag(Sinv[p.index]))
    return np.array(rows)


def paired_back_matrix(S, pairs):
    """Real (Q x 2P) matrix mapping (re, im) rows of the block solutions back to the real stage
    vector k = S z (the conjugate partner's column contributes the complex conjugate)."""
    Q = S.shape[0]
    cols = []
    for p in pairs:
        s = S[:, p.index]
        if p.is_real:
            cols.append(np.real(s))
            cols.append(np.zeros(Q))
        else:
            cols.append(2.0 * np.real(s))
            cols.append(-2.0 * np.imag(s))
    return np.array(cols).T
