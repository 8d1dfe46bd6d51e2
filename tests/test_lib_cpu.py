"""C-ABI library: loads, exports every symbol include/spk.h declares, host-side setup is right
(no GPU needed)."""

import os
import re

import numpy as np
import pytest

from oracle.fem_qk import Hierarchy, prolongation_1d
from paper_2209_06700_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "spk.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(spk_\w+)\(", text, re.M)))


def test_library_exports_header():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) > 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.EXPORTED, f"{s} has no ctypes signature"


def test_version_and_errors():
    lib = _lib.load()
    assert lib.spk_version() == 1
    ctx = _lib.c_vp()
    rc = lib.spk_ctx_create(4, 2, 1, _lib.ctypes.byref(ctx))
    assert rc == 2 and b"dim" in lib.spk_last_error()
    rc = lib.spk_ctx_create(3, 2, 7, _lib.ctypes.byref(ctx))
    assert rc == 7


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_host_tables_match_oracle(k):
    from paper_2209_06700_b200.fem import build_hierarchy

    h = build_hierarchy(3, 3, k)
    o = Hierarchy(3, 3, k)
    for L in range(4):
        assert h.levels[L].n_per_axis == o.levels[L].n_per_axis
        assert np.allclose(h.levels[L].nodes_1d, o.levels[L].coords, atol=1e-15, rtol=0)
        assert np.allclose(h.levels[L].elem_mass, o.levels[L].elem_mass, rtol=1e-14, atol=0)
        assert np.allclose(h.levels[L].elem_stiffness, o.levels[L].elem_stiffness, rtol=1e-13, atol=0)
        assert np.allclose(h.operator_diagonal(L, 1.5, 0.1), o.operator_diagonal(L, 1.5, 0.1), rtol=1e-14)
    assert np.allclose(h.prolong_table, prolongation_1d(k, 1)[:, : k + 1], atol=1e-15)


def test_hierarchy_guards():
    from paper_2209_06700_b200.errors import ConfigurationError
    from paper_2209_06700_b200.fem import build_hierarchy

    with pytest.raises(ConfigurationError):
        build_hierarchy(4, 2)
    with pytest.raises(ConfigurationError):
        build_hierarchy(2, 0)
    with pytest.raises(ConfigurationError):
        build_hierarchy(2, 8)
    with pytest.raises(ConfigurationError):
        build_hierarchy(2, 2, degree=5)


def test_slab_window_host_side():
    """spk_ctx_set_slab: validation and the local level sizes the Python slab layout relies on."""
    from paper_2209_06700_b200.slab import SlabPartition

    lib = _lib.load()
    k, L, B = 2, 4, 4
    ctx = _lib.c_vp()
    assert lib.spk_ctx_create(3, L, k, _lib.ctypes.byref(ctx)) == 0
    try:
        for b in range(B):
            part = SlabPartition(k, L, B, b)
            for level in part.dist_levels:
                w = part.window(level)
                rc = lib.spk_ctx_set_slab(ctx, level, w.x_elems, w.x0, 2, w.x_elems, 1 if w.last else 0)
                assert rc == 0, lib.spk_last_error()
                npa, nd, hh, ne = _lib.c_int(), _lib.c_ll(), _lib.c_dbl(), _lib.c_int()
                assert lib.spk_level_info(ctx, level, _lib.ctypes.byref(npa), _lib.ctypes.byref(nd),
                                          _lib.ctypes.byref(hh), _lib.ctypes.byref(ne)) == 0
                assert nd.value == w.local_numel and npa.value == w.nax
        # invalid windows: elements past the mesh, misaligned offset, empty range
        assert lib.spk_ctx_set_slab(ctx, L, 4, k * 14, 2, 4, 1) == 2
        assert lib.spk_ctx_set_slab(ctx, L, 4, 1, 2, 4, 0) == 2
        assert lib.spk_ctx_set_slab(ctx, L, 4, 0, 3, 3, 0) == 2
        assert lib.spk_set_cheb_split(ctx, 0) == 0 and lib.spk_set_vsplit(ctx, 0) == 0
    finally:
        lib.spk_ctx_destroy(ctx)
