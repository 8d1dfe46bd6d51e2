"""Race / barrier checks without compute-sanitizer (it is closed on this GPU pool): the kernels with
inter-thread or inter-CTA synchronisation -- the cooperative MGS column (grid barriers, partials
summed in CTA order), the single-CTA fused coarse V-cycle (shared-memory levels, CTA barriers), K1's
plane pipeline (one barrier per plane) -- must be bitwise run-to-run deterministic; a missing barrier
or a data race shows up as run-to-run differences under repetition with other work in between."""

import numpy as np
import pytest
import torch

from paper_2209_06700_b200 import _lib
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.krylov import _ctx
from paper_2209_06700_b200.multigrid import MultiBlockSolver, VCycleConfig

pytestmark = pytest.mark.gpu


def test_coarse_vcycle_and_k1_bitwise_repeatable():
    h = build_hierarchy(3, 4, 2)
    mb = MultiBlockSolver(h, [3.2, 2.1, 9.0], 0.01, VCycleConfig(smoother_degree=3))
    g = torch.Generator(device="cuda").manual_seed(5)
    b = torch.rand((3, h.levels[4].n_dofs), dtype=torch.float64, device="cuda", generator=g)
    ref = mb.apply_device(b).clone()
    assert mb._cv_level >= 1  # the fused single-CTA coarse V-cycle is on this path
    u = torch.rand((3, h.levels[4].n_dofs), dtype=torch.float64, device="cuda", generator=g)
    DM, DK = np.eye(3), 1e-2 * np.arange(1.0, 10.0).reshape(3, 3)
    vref = h.apply_stage_operator(4, DM, DK, u).clone()
    noise = torch.empty(1 << 22, dtype=torch.float64, device="cuda")
    for i in range(10):
        noise.normal_()  # other work on the device between repetitions
        assert torch.equal(mb.apply_device(b), ref), i
        assert torch.equal(h.apply_stage_operator(4, DM, DK, u), vref), i


@pytest.mark.parametrize("n,j", [(5000, 6), (1 << 20, 6), (1 << 20, 5), ((1 << 25) + 9, 6), ((1 << 25) + 9, 3)])
def test_mgs_column_bitwise_repeatable(n, j):
    # (n <= 2^25: the cooperative single-launch column; above: the paired sweeps of mgs2_kernel. The
    # basis here is NOT orthogonal, so the paired form's correction h_b = s_b - h_a <v_a, v_b> is
    # exercised with a large mutual dot; odd and even numbers of basis vectors)
    g = torch.Generator(device="cuda").manual_seed(6)
    basis = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(j + 1)]
    w0 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    ptrs = (_lib.ctypes.c_void_p * (j + 1))(*[b.data_ptr() for b in basis])
    from paper_2209_06700_b200._device import stream_ptr
    outs = []
    for _ in range(6):
        w = w0.clone()
        hcol = torch.zeros(j + 2, dtype=torch.float64, device="cuda")
        vn = torch.empty_like(w)
        _lib.call("spk_mgs_column", _ctx(), n, j, _lib.ctypes.addressof(ptrs), w.data_ptr(), hcol.data_ptr(),
                  vn.data_ptr(), stream_ptr(w.device))
        outs.append((hcol.clone(), vn.clone()))
    for hc, vn in outs[1:]:
        assert torch.equal(hc, outs[0][0]) and torch.equal(vn, outs[0][1])
    # and the column equals modified Gram-Schmidt in float64 on the host to rounding
    W = w0.cpu().numpy().copy()
    B = [b.cpu().numpy() for b in basis]
    h = []
    for i in range(j + 1):
        h.append(B[i] @ W)
        W = W - h[-1] * B[i]
    h.append(np.linalg.norm(W))
    np.testing.assert_allclose(outs[0][0].cpu().numpy(), h, rtol=1e-11, atol=1e-11 * abs(h[0]))
