"""Windowed K1 launches: x-slab partition (2 ranks emulated on one GPU with a manual halo copy) and
the chunked host pipeline reproduce the full operator (separable inputs give exact 1D answers)."""

import numpy as np
import pytest
import torch

from paper_2209_06700_b200 import _lib
from paper_2209_06700_b200._device import ptr
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.parallel import SlabLayout
from paper_2209_06700_b200.pipeline import HostStageOperator
from paper_2209_06700_b200.tableau import radau_iia

pytestmark = pytest.mark.gpu


def assemble(elem, E, k):
    n = k * E + 1
    m = np.zeros((n, n))
    for e in range(E):
        m[k * e : k * e + k + 1, k * e : k * e + k + 1] += elem
    return m


@pytest.mark.parametrize("k,L,Q", [(2, 3, 2), (4, 2, 3), (1, 4, 4)])
def test_two_slab_emulation(cuda, k, L, Q):
    h = build_hierarchy(3, L, k)
    lvl = h.levels[L]
    E, nax = lvl.n_elements, lvl.n_per_axis
    world = 2
    NX = k * E * world + 1  # global planes along x
    rng = np.random.default_rng(4)
    ax = rng.standard_normal(NX)
    ay, az = rng.standard_normal(nax), rng.standard_normal(nax)
    coef = rng.standard_normal(Q)
    A = radau_iia(Q).A
    DM, DK = np.eye(Q), 1e-2 * A
    Mx, Kx = assemble(lvl.elem_mass, E * world, k), assemble(lvl.elem_stiffness, E * world, k)
    My, Ky = lvl.mass_1d, lvl.stiffness_1d
    sep = lambda a, b, c: np.multiply.outer(np.multiply.outer(a, b), c)
    Mu = sep(Mx @ ax, My @ ay, My @ az)
    Ku = sep(Kx @ ax, My @ ay, My @ az) + sep(Mx @ ax, Ky @ ay, My @ az) + sep(Mx @ ax, My @ ay, Ky @ az)
    ref = np.einsum("i,xyz->ixyz", DM @ coef, Mu) + np.einsum("i,xyz->ixyz", DK @ coef, Ku)
    glob = np.einsum("i,xyz->ixyz", coef, sep(ax, ay, az))
    plane = nax * nax
    for rank in range(world):
        lay = SlabLayout(k, E, plane, world, rank)
        buf = np.zeros((Q, lay.nplanes, nax, nax))
        g0 = rank * k * E - k  # global plane of local plane 0
        for p in range(lay.nplanes):
            gp = g0 + p
            if 0 <= gp < NX and (rank > 0 or p >= k):
                buf[:, p] = glob[:, gp]
        u = torch.from_numpy(buf.reshape(Q, -1)).cuda()
        v = torch.zeros_like(u)
        n = lay.local_numel
        DMc, DKc = np.ascontiguousarray(DM), np.ascontiguousarray(DK)
        if rank == 0:
            bu, bv = u[:, k * plane :], v[:, k * plane :]
            xe, eb, ee = E, 0, E
        else:
            bu, bv, xe, eb, ee = u, v, E + 1, 1, E + 1
        _lib.call("spk_stage_apply_slab", h.ctx, L, Q, DMc.ctypes.data_as(_lib.P_dbl),
                  DKc.ctypes.data_as(_lib.P_dbl), ptr(bu), n, ptr(bv), n, xe, eb, ee,
                  1 if rank == world - 1 else 0, torch.cuda.current_stream().cuda_stream)
        out = v.cpu().numpy().reshape(Q, lay.nplanes, nax, nax)
        for p in range(lay.n_owned_planes):
            gp = rank * k * E + p
            err = np.abs(out[:, k + p] - ref[:, gp]).max() / np.abs(ref).max()
            assert err < 1e-12, (rank, p, err)


def test_host_pipeline_matches_device_apply(cuda):
    h = build_hierarchy(3, 4, 4)
    L = 4
    Q = 3
    DM, DK = np.eye(Q), 1e-3 * radau_iia(Q).A
    n = h.levels[L].n_dofs
    u = torch.rand((Q, n), dtype=torch.float64) * 2 - 1
    u_host = u.pin_memory()
    v_host = torch.empty_like(u_host).pin_memory()
    op = HostStageOperator(h, L, DM, DK, chunks=5)
    op.apply(u_host, v_host)
    torch.cuda.synchronize()
    ref = h.apply_stage_operator(L, DM, DK, u.cuda()).cpu()
    assert torch.equal(v_host, ref)
