"""ctypes binding of libspk (`_spk.so`, the C-ABI declared in include/spk.h).

There is no fallback: if the shared library is missing or a CUDA device is absent when a device
entry point is called, the call raises. Error codes are mapped onto the reference package's
exception taxonomy (errors.py).
"""

import ctypes
import os

from .errors import (
    CommunicationError,
    ConfigurationError,
    DimensionMismatchError,
    NumericalFailureError,
    SpectralFailureError,
    UnsupportedDegreeError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPK_LIB_PATH", os.path.join(_HERE, "_spk.so"))

c_int = ctypes.c_int
c_ll = ctypes.c_longlong
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P_dbl = ctypes.POINTER(c_dbl)

_SIGS = {
    "spk_version": ([], c_int),
    "spk_last_error": ([], ctypes.c_char_p),
    "spk_ctx_create": ([c_int, c_int, c_int, ctypes.POINTER(c_vp)], c_int),
    "spk_ctx_destroy": ([c_vp], c_int),
    "spk_ctx_set_slab": ([c_vp, c_int, c_int, c_int, c_int, c_int, c_int], c_int),
    "spk_level_info": ([c_vp, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_ll), P_dbl,
                        ctypes.POINTER(c_int)], c_int),
    "spk_level_tables": ([c_vp, c_int, P_dbl, P_dbl], c_int),
    "spk_nodes_1d": ([c_vp, c_int, P_dbl], c_int),
    "spk_prolong_table": ([c_vp, P_dbl], c_int),
    "spk_apply_smem": ([c_int, c_int], c_int),
    "spk_set_chunks": ([c_vp, c_int], c_int),
    "spk_stage_apply": ([c_vp, c_int, c_int, P_dbl, P_dbl, c_int, c_vp, c_ll, c_vp, c_ll, c_vp], c_int),
    "spk_stage_apply_slab": ([c_vp, c_int, c_int, P_dbl, P_dbl, c_vp, c_ll, c_vp, c_ll, c_int, c_int, c_int,
                              c_int, c_vp], c_int),
    "spk_block_apply": ([c_vp, c_int, c_int, P_dbl, c_int, c_dbl, c_int, c_vp, c_ll, c_vp, c_ll, c_vp],
                        c_int),
    "spk_pair_apply": ([c_vp, c_int, c_dbl, c_dbl, c_dbl, c_int, c_vp, c_vp, c_vp], c_int),
    "spk_residual": ([c_vp, c_int, c_int, P_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, P_dbl, c_vp], c_int),
    "spk_cheb_init": ([c_vp, c_int, c_int, P_dbl, c_dbl, P_dbl, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_cheb_step": ([c_vp, c_int, c_int, P_dbl, c_dbl, P_dbl, P_dbl, c_vp, c_vp, c_vp, c_vp, c_int, c_vp,
                       c_vp], c_int),
    "spk_cheb_start": ([c_vp, c_int, c_int, P_dbl, c_dbl, P_dbl, c_vp, c_vp, c_vp], c_int),
    "spk_cheb_first_step": ([c_vp, c_int, c_int, P_dbl, c_dbl, P_dbl, P_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_int,
                             c_vp, c_vp], c_int),
    "spk_cheb_split": ([c_vp, c_int, c_int], c_int),
    "spk_set_cheb_split": ([c_vp, c_ll], c_int),
    "spk_set_vsplit": ([c_vp, c_int], c_int),
    "spk_pair_residual": ([c_vp, c_int, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp], c_int),
    "spk_pair_cheb_init": ([c_vp, c_int, c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_pair_cheb_step": ([c_vp, c_int, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_int,
                            c_vp, c_vp], c_int),
    "spk_dinv_norm": ([c_vp, c_int, c_int, c_dbl, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_transfer": ([c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_int, c_vp], c_int),
    "spk_axpy_flag": ([c_ll, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_combine": ([c_vp, c_int, c_ll, c_int, c_int, P_dbl, c_vp, c_ll, c_vp, c_ll, c_int, c_vp], c_int),
    "spk_peer_combine": ([c_ll, c_int, c_vp, c_int, P_dbl, c_vp, c_ll, c_int, c_vp], c_int),
    "spk_ipc_alloc": ([c_ll, ctypes.POINTER(c_vp), c_vp], c_int),
    "spk_ipc_open": ([c_vp, ctypes.POINTER(c_vp)], c_int),
    "spk_ipc_close": ([c_vp], c_int),
    "spk_ipc_free": ([c_vp], c_int),
    "spk_copy_d2d": ([c_vp, c_vp, c_ll, c_vp], c_int),
    "spk_mgs": ([c_vp, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_mgs_partial": ([c_vp, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_sqrt_dev": ([c_vp, c_int, c_vp], c_int),
    "spk_fp64_probe": ([c_int, c_int, c_int, c_vp, c_vp], c_int),
    "spk_givens": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp], c_int),
    "spk_band_axis": ([c_ll, c_int, c_int, c_ll, c_vp, c_vp, c_int, c_vp, c_vp, c_int, c_vp], c_int),
    "spk_gauss_l2": ([c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp, c_vp], c_int),
    "spk_scale_div": ([c_ll, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_mgs_column": ([c_vp, c_ll, c_int, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_coarse_vcycle_level": ([c_vp], c_int),
    "spk_coarse_vcycle": ([c_vp, c_int, c_int, P_dbl, c_dbl, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
                          c_int),
    "spk_lincomb": ([c_ll, c_int, c_vp, c_vp, c_vp, c_vp], c_int),
    "spk_outer3": ([c_vp, c_int, c_vp, c_vp, c_vp], c_int),
    "spk_rhs": ([c_vp, c_int, c_int, c_vp, P_dbl, P_dbl, c_vp, c_vp, c_vp], c_int),
    "spk_update": ([c_ll, c_int, c_vp, c_vp, c_dbl, c_vp, c_vp], c_int),
    "spk_mask": ([c_vp, c_int, c_int, c_vp, c_dbl, c_vp], c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load `_spk.so` (raises if it has not been built; there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libspk not built ({LIB_PATH} missing): run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    lax = os.environ.get("SPK_LIB_LAX") == "1"  # A/B of older library builds (tools/ab_apply.py)
    for name, (args, res) in _SIGS.items():
        if lax and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


_ERRORS = {
    1: DimensionMismatchError,
    2: ConfigurationError,
    3: NumericalFailureError,
    4: SpectralFailureError,
    5: RuntimeError,
    6: CommunicationError,
    7: UnsupportedDegreeError,
}


def check(rc):
    if rc != 0:
        msg = load().spk_last_error().decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def dbl_array(values):
    vals = [float(v) for v in values]
    return (c_dbl * max(1, len(vals)))(*vals)
