"""Device-resident nested uniform grids with Q_k Lagrange elements on [0,1]^dim.

Drop-in mirror of the reference fem module (GridHierarchy fem.py:72-273, build_hierarchy :300,
manufactured :305, HeatProblem :342) generalised to degree k = 1..4 on Gauss-Lobatto-Legendre
nodes, with the operator actions executed by libspk's sm_100a kernels:

  apply_mass / apply_stiffness / apply_shifted / apply_constrained  -> spk_block_apply (K1, block mode)
  apply_stage_operator (D_M (x) M + D_K (x) K)                       -> spk_stage_apply (K1, coupled)
  prolong / restrict                                                 -> spk_transfer

Inputs may be torch CUDA tensors (results stay on the device) or numpy arrays (copied in and out,
for callers written against the reference). At k = 1 every operator reproduces the reference
(pinned against its golden vectors in tests/).
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import is_host, like_input, ptr, require_cuda, stream_ptr, to_device
from .errors import ConfigurationError, DimensionMismatchError

_DEFERRED_CTX = []  # contexts collected during a CUDA graph capture, destroyed at the next chance

MAX_DEGREE = 4


def _gauss01(m):
    x, w = np.polynomial.legendre.leggauss(m)
    return 0.5 * (x + 1.0), 0.5 * w


def _lagrange(nodes, a, x):
    v = np.ones_like(np.asarray(x, dtype=float))
    for m, xm in enumerate(nodes):
        if m != a:
            v = v * (x - xm) / (nodes[a] - xm)
    return v


@dataclass
class GridLevel:
    """One refinement level: 2^index elements per axis, k*2^index + 1 nodes per axis."""

    index: int
    dim: int
    degree: int
    n_per_axis: int
    h: float
    nodes_1d: np.ndarray
    elem_mass: np.ndarray       # (k+1, k+1), scaled by h
    elem_stiffness: np.ndarray  # (k+1, k+1), scaled by 1/h
    interior_mask: np.ndarray   # flat bool, True on interior DoFs
    _dense: dict = field(default_factory=dict, repr=False)

    @property
    def shape(self):
        return (self.n_per_axis,) * self.dim

    @property
    def n_dofs(self):
        return self.n_per_axis ** self.dim

    @property
    def n_elements(self):
        return 2 ** self.index

    @property
    def n_cells(self):
        return self.n_elements ** self.dim

    def axis_coords(self):
        return self.nodes_1d.copy()

    def _assemble(self, elem):
        k, n = self.degree, self.n_per_axis
        m = np.zeros((n, n))
        for e in range(self.n_elements):
            m[k * e : k * e + k + 1, k * e : k * e + k + 1] += elem
        return m

    @property
    def mass_1d(self):
        """Assembled 1D mass matrix (host, dense; for inspection only)."""
        if "M" not in self._dense:
            self._dense["M"] = self._assemble(self.elem_mass)
        return self._dense["M"]

    @property
    def stiffness_1d(self):
        if "K" not in self._dense:
            self._dense["K"] = self._assemble(self.elem_stiffness)
        return self._dense["K"]

    def diag_1d(self):
        return np.diag(self.mass_1d).copy(), np.diag(self.stiffness_1d).copy()


class GridHierarchy:
    """Nested grids, levels 0..max_level, with device operator actions."""

    def __init__(self, dim, max_level, degree=1, device=None):
        if dim not in (1, 2, 3):
            raise ConfigurationError(f"dim must be 1, 2 or 3, got {dim}")
        if not (1 <= max_level <= 7):
            raise ConfigurationError(f"max_level must be in [1, 7], got {max_level}")
        if not (1 <= degree <= MAX_DEGREE):
            raise ConfigurationError(f"degree must be in [1, {MAX_DEGREE}], got {degree}")
        self.dim = dim
        self.max_level = max_level
        self.degree = degree
        lib = _lib.load()
        ctx = _lib.c_vp()
        _lib.check(lib.spk_ctx_create(dim, max_level, degree, _lib.ctypes.byref(ctx)))
        self._ctx = ctx
        self._device = torch.device(device) if device is not None else None
        k = degree
        self.levels = []
        for ell in range(max_level + 1):
            npa = _lib.c_int()
            nd = _lib.c_ll()
            h = _lib.c_dbl()
            ne = _lib.c_int()
            _lib.check(lib.spk_level_info(ctx, ell, _lib.ctypes.byref(npa), _lib.ctypes.byref(nd),
                                          _lib.ctypes.byref(h), _lib.ctypes.byref(ne)))
            n = npa.value
            nodes = np.zeros(n)
            _lib.check(lib.spk_nodes_1d(ctx, ell, nodes.ctypes.data_as(_lib.P_dbl)))
            Me = np.zeros((k + 1, k + 1))
            Ke = np.zeros((k + 1, k + 1))
            _lib.check(lib.spk_level_tables(ctx, ell, Me.ctypes.data_as(_lib.P_dbl),
                                            Ke.ctypes.data_as(_lib.P_dbl)))
            inter = np.ones(n, dtype=bool)
            inter[0] = inter[-1] = False
            mask = inter
            for _ in range(dim - 1):
                mask = np.logical_and.outer(mask, inter)
            self.levels.append(GridLevel(ell, dim, k, n, h.value, nodes, Me, Ke, mask.ravel()))
        P = np.zeros((2 * k + 1, k + 1))
        _lib.check(lib.spk_prolong_table(ctx, P.ctypes.data_as(_lib.P_dbl)))
        self.prolong_table = P
        self._masks = {}
        self._scratch = {}

    def __del__(self):
        try:
            if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
                _DEFERRED_CTX.append(self._ctx)  # no cudaFree inside a graph capture
                return
            _lib.load().spk_ctx_destroy(self._ctx)
            while _DEFERRED_CTX:
                _lib.load().spk_ctx_destroy(_DEFERRED_CTX.pop())
        except Exception:
            pass

    # ---- basic properties (reference fem.py:104-110) ----
    @property
    def finest(self):
        return self.levels[-1]

    @property
    def n(self):
        return self.finest.n_dofs

    @property
    def device(self):
        if self._device is None:
            require_cuda()
            self._device = torch.device("cuda", torch.cuda.current_device())
        return self._device

    @property
    def ctx(self):
        return self._ctx

    def mask_tensor(self, level):
        if level not in self._masks:
            self._masks[level] = torch.from_numpy(self.levels[level].interior_mask).to(self.device)
        return self._masks[level]

    def scratch(self, key, numel):
        buf = self._scratch.get(key)
        if buf is None or buf.numel() < numel:
            buf = torch.empty(numel, dtype=torch.float64, device=self.device)
            self._scratch[key] = buf
        return buf

    def _check(self, level, u):
        lvl = self.levels[level]
        if u.shape[-1] != lvl.n_dofs:
            raise DimensionMismatchError(f"level {level} expects {lvl.n_dofs} DoFs, got {u.shape[-1]}")
        return lvl

    def _prep(self, level, u):
        """(device tensor viewed as (nblk, n), leading shape, original container)."""
        self._check(level, u)
        lead = tuple(u.shape[:-1])
        d = to_device(u, self.device)
        n = self.levels[level].n_dofs
        return d.reshape(-1, n), lead

    # ---- operator actions ----
    def apply_block(self, level, lams, tau, u, constrained=False, out=None):
        """Device core: out_b = lams_b M u_b + tau K u_b for u of shape (nblk, n) (device)."""
        nblk, n = u.shape
        if out is None:
            out = torch.empty_like(u)
        lams = np.atleast_1d(np.asarray(lams, dtype=float))
        uniform = 1 if lams.size == 1 else 0
        if not uniform and lams.size != nblk:
            raise DimensionMismatchError(f"{lams.size} shifts for {nblk} blocks")
        _lib.call("spk_block_apply", self._ctx, level, nblk, _lib.dbl_array(lams), uniform, float(tau),
                  1 if constrained else 0, ptr(u), n, ptr(out), n, stream_ptr(self.device))
        return out

    def _shifted(self, level, lam, tau, u, constrained):
        u2, lead = self._prep(level, u)
        lam_arr = np.asarray(lam, dtype=float)
        if lam_arr.ndim > 0 and lam_arr.size > 1:
            lam_arr = np.broadcast_to(lam_arr.reshape(-1, *([1] * max(0, len(lead) - 1))),
                                      lead).reshape(-1)
        v = self.apply_block(level, lam_arr, tau, u2, constrained)
        return like_input(v.reshape(*lead, -1), u)

    def apply_mass(self, level, u):
        """v = M u, unconstrained, for (..., n) stacked vectors (reference fem.py:120-128)."""
        return self._shifted(level, 1.0, 0.0, u, False)

    def apply_stiffness(self, level, u):
        """v = K u, unconstrained (reference fem.py:130-143)."""
        return self._shifted(level, 0.0, 1.0, u, False)

    def apply_shifted(self, level, lam, tau, u):
        """v = (lam M + tau K) u; lam scalar or per leading block (reference fem.py:145-151)."""
        return self._shifted(level, lam, tau, u, False)

    def apply_constrained(self, level, lam, tau, u):
        """Interior rows (lam M + tau K) on the masked input, identity on boundary rows
        (reference fem.py:160-170)."""
        return self._shifted(level, lam, tau, u, True)

    def apply_stage_operator(self, level, DM, DK, u, constrained=False, out=None):
        """K1: v_i = sum_j (DM_ij M + DK_ij K) u_j on (Q, n) stage vectors in one launch."""
        u2, lead = self._prep(level, u)
        Q, n = u2.shape
        DM = np.ascontiguousarray(np.asarray(DM, dtype=float).reshape(Q, Q))
        DK = np.ascontiguousarray(np.asarray(DK, dtype=float).reshape(Q, Q))
        if out is None:
            out = torch.empty_like(u2)
        if Q <= 4:
            _lib.call("spk_stage_apply", self._ctx, level, Q, DM.ctypes.data_as(_lib.P_dbl),
                      DK.ctypes.data_as(_lib.P_dbl), 1 if constrained else 0, ptr(u2), n, ptr(out), n,
                      stream_ptr(self.device))
        else:
            # Q > 4: per-stage M u_j and K u_j in block launches, then the (D (x) I) combines
            mu = self.apply_block(level, 1.0, 0.0, u2, constrained)
            ku = self.apply_block(level, 0.0, 1.0, u2, constrained)
            from .tensor_ops import dense_combine
            dense_combine(DM, mu, out=out, hierarchy=self)
            dense_combine(DK, ku, out=out, accumulate=True, hierarchy=self)
            if constrained:
                m = self.mask_tensor(level)
                out.copy_(torch.where(m, out, u2))
        return like_input(out.reshape(*lead, -1), u)

    def constrain(self, level, vec, boundary_values=0.0):
        """Copy of vec with boundary DoFs overwritten (reference fem.py:153-158)."""
        d, lead = self._prep(level, vec)
        out = d.clone()
        _lib.call("spk_mask", self._ctx, level, out.shape[0], ptr(out), float(boundary_values),
                  stream_ptr(self.device))
        return like_input(out.reshape(*lead, -1), vec)

    def operator_diagonal(self, level, lam, tau):
        """diag(lam M + tau K), 1.0 on constrained rows (reference fem.py:172-187)."""
        lvl = self.levels[level]
        dm1, dk1 = lvl.diag_1d()
        dm = dm1
        for _ in range(self.dim - 1):
            dm = np.multiply.outer(dm, dm1)
        dk = np.zeros(lvl.shape)
        for d in range(self.dim):
            term = np.ones(())
            for ax in range(self.dim):
                term = np.multiply.outer(term, dk1 if ax == d else dm1)
            dk = dk + term
        diag = (lam * dm + tau * dk).ravel()
        return np.where(lvl.interior_mask, diag, 1.0)

    # ---- transfers ----
    def prolong_into(self, coarse_level, uc, out, accumulate=False):
        """out (nblk, n_fine) (+)= P uc on device."""
        nblk = uc.shape[0]
        nf = self.levels[coarse_level + 1].n_dofs
        scr = self.scratch(("transfer", nblk), 2 * nblk * nf)
        _lib.call("spk_transfer", self._ctx, coarse_level + 1, nblk, 1, ptr(uc), ptr(out), ptr(scr),
                  1 if accumulate else 0, 0, stream_ptr(self.device))
        return out

    def restrict_into(self, fine_level, rf, out, mask=False):
        nblk = rf.shape[0]
        nf = self.levels[fine_level].n_dofs
        scr = self.scratch(("transfer", nblk), 2 * nblk * nf)
        _lib.call("spk_transfer", self._ctx, fine_level, nblk, 0, ptr(rf), ptr(out), ptr(scr), 0,
                  1 if mask else 0, stream_ptr(self.device))
        return out

    def prolong(self, coarse_level, u_coarse):
        """Q_k embedding interpolation from level l to l+1 (reference fem.py:189-199)."""
        d, lead = self._prep(coarse_level, u_coarse)
        out = torch.empty((d.shape[0], self.levels[coarse_level + 1].n_dofs), dtype=torch.float64,
                          device=self.device)
        self.prolong_into(coarse_level, d, out)
        return like_input(out.reshape(*lead, -1), u_coarse)

    def restrict(self, fine_level, r_fine):
        """Transpose of prolongation, level l to l-1 (reference fem.py:201-211)."""
        d, lead = self._prep(fine_level, r_fine)
        out = torch.empty((d.shape[0], self.levels[fine_level - 1].n_dofs), dtype=torch.float64,
                          device=self.device)
        self.restrict_into(fine_level, d, out)
        return like_input(out.reshape(*lead, -1), r_fine)

    # ---- geometry, load vector, error ----
    def node_coords(self, level):
        """(n_dofs, dim) node coordinates in C order (reference fem.py:213-218)."""
        axes = [self.levels[level].nodes_1d] * self.dim
        mesh = np.meshgrid(*axes, indexing="ij")
        return np.stack([m.ravel() for m in mesh], axis=-1)

    def _gauss_axis(self, level):
        lvl = self.levels[level]
        k, N, h = self.degree, lvl.n_elements, lvl.h
        xg, wg = _gauss01(k + 1)
        pts = ((np.arange(N)[:, None] + xg[None, :]) * h).ravel()
        ref_nodes = self.levels[0].nodes_1d  # level 0 is the reference element [0, 1]
        shape = np.stack([_lagrange(ref_nodes, a, xg) for a in range(k + 1)])  # (nodes, gauss)
        return pts, xg, wg, shape

    def load_matrix_1d(self, level):
        """(n_ax, N(k+1)) map from Gauss-point values (x weight) to nodal load contributions."""
        lvl = self.levels[level]
        k, N, h = self.degree, lvl.n_elements, lvl.h
        _, xg, wg, shape = self._gauss_axis(level)
        B = np.zeros((lvl.n_per_axis, N * (k + 1)))
        for e in range(N):
            for a in range(k + 1):
                B[k * e + a, (k + 1) * e : (k + 1) * (e + 1)] += shape[a] * wg * h
        return B

    def interp_matrix_1d(self, level):
        """(N(k+1), n_ax) nodal -> Gauss-point interpolation."""
        lvl = self.levels[level]
        k, N = self.degree, lvl.n_elements
        _, _, _, shape = self._gauss_axis(level)
        I = np.zeros((N * (k + 1), lvl.n_per_axis))
        for e in range(N):
            for a in range(k + 1):
                I[(k + 1) * e : (k + 1) * (e + 1), k * e + a] = shape[a]
        return I

    def _band_dev(self, key, mat):
        """Device (col0, vals, bw) of a banded host matrix, cached per (kind, level)."""
        cache = self.__dict__.setdefault("_bands", {})
        ent = cache.get(key)
        if ent is None:
            nz = mat != 0.0
            first = np.where(nz.any(axis=1), nz.argmax(axis=1), 0)
            last = np.where(nz.any(axis=1), mat.shape[1] - 1 - nz[:, ::-1].argmax(axis=1), 0)
            bw = int(max(1, (last - first + 1).max()))
            col0 = np.minimum(first, mat.shape[1] - bw).astype(np.int32)
            vals = np.take_along_axis(mat, col0[:, None] + np.arange(bw)[None, :], axis=1)
            ent = (torch.from_numpy(col0).to(self.device), torch.from_numpy(np.ascontiguousarray(vals)).to(self.device),
                   bw, mat.shape[1], mat.shape[0])
            cache[key] = ent
        return ent

    def _axes_apply(self, key, mat, arr):
        """mat applied along every axis of the (nin,)*dim device array (spk_band_axis per axis)."""
        col0, vals, bw, nin, nout = self._band_dev(key, mat)
        st = stream_ptr(self.device)
        cur = arr.contiguous()
        for ax in range(self.dim):
            shp = list(cur.shape)
            A = int(np.prod(shp[:ax], dtype=np.int64))
            B = int(np.prod(shp[ax + 1 :], dtype=np.int64))
            shp[ax] = nout
            out = torch.empty(shp, dtype=torch.float64, device=self.device)
            _lib.call("spk_band_axis", A, nin, nout, B, ptr(col0), ptr(vals), bw, ptr(cur), ptr(out), 0, st)
            cur = out
        return cur

    def _gauss_points(self, level):
        pts1, _, _, _ = self._gauss_axis(level)
        mesh = np.meshgrid(*([pts1] * self.dim), indexing="ij")
        return pts1, np.stack([m.ravel() for m in mesh], axis=-1)

    def load_vector_device(self, level, f, t):
        """Device (n,) consistent load vector int f(x,t) phi_i, (k+1)-point Gauss rule per axis
        (reference fem.py:220-246). Separable sources (SeparableSolution, and the reference's
        `manufactured()` family, which carry `.separable`) are formed on the device from the 1D
        load vector (spk_outer3, times F(t)); general callables are evaluated on the host at the
        tensor Gauss points (they are user numpy code) and contracted by the device Gauss-to-node
        kernel (spk_band_axis along each axis)."""
        sep = getattr(f, "separable", None)
        if sep is not None:
            g1 = torch.from_numpy(self.load_vector_1d(level, sep.s)).to(self.device)
            out = torch.empty(self.levels[level].n_dofs, dtype=torch.float64, device=self.device)
            _lib.call("spk_outer3", self._ctx, level, ptr(g1), ptr(out), stream_ptr(self.device))
            return out.mul_(float(sep.F(t)))
        pts1, pts = self._gauss_points(level)
        fv = torch.from_numpy(np.ascontiguousarray(np.asarray(f(pts, t), dtype=float))).to(self.device)
        out = self._axes_apply(("load", level), self.load_matrix_1d(level), fv.reshape((pts1.size,) * self.dim))
        return out.reshape(-1)

    def load_vector(self, level, f, t):
        """Host (numpy) load vector, as the reference returns it (fem.py:220-246); the arithmetic
        runs on the device (load_vector_device)."""
        return self.load_vector_device(level, f, t).cpu().numpy()

    def load_vector_1d(self, level, s):
        """1D load vector of a spatial factor s(x) (separable sources: F = prod_a g[i_a])."""
        pts1, _, _, _ = self._gauss_axis(level)
        return self.load_matrix_1d(level) @ np.asarray(s(pts1), dtype=float)

    def l2_error(self, level, u_nodal, u_exact, t):
        """L2 norm of u_h - u_exact by per-cell (k+1)^dim Gauss quadrature (reference fem.py:248-273):
        u_h interpolated to the tensor Gauss points on the device (spk_band_axis), then one fused
        weighted-square reduction (spk_gauss_l2) with u_exact evaluated in the kernel for separable
        solutions or taken from host evaluation at the Gauss points otherwise."""
        lvl = self.levels[level]
        pts1, _, wg, _ = self._gauss_axis(level)
        u = to_device(u_nodal, self.device).reshape(lvl.shape)
        ug = self._axes_apply(("interp", level), self.interp_matrix_1d(level), u)
        w1 = torch.from_numpy(np.tile(wg * lvl.h, lvl.n_elements)).to(self.device)
        out = torch.empty(1, dtype=torch.float64, device=self.device)
        sep = getattr(u_exact, "separable", None)
        st = stream_ptr(self.device)
        if sep is not None:
            s1 = torch.from_numpy(np.asarray(sep.s(pts1), dtype=float)).to(self.device)
            _lib.call("spk_gauss_l2", self._ctx, self.dim, pts1.size, ptr(ug), ptr(w1), None, ptr(s1),
                      float(sep.T(t)), ptr(out), st)
        else:
            _, pts = self._gauss_points(level)
            ue = torch.from_numpy(np.ascontiguousarray(np.asarray(u_exact(pts, t), dtype=float))).to(self.device)
            _lib.call("spk_gauss_l2", self._ctx, self.dim, pts1.size, ptr(ug), ptr(w1), ptr(ue), None, 0.0,
                      ptr(out), st)
        return float(out.item())


def build_hierarchy(dim, max_level, degree=1, device=None):
    """Nested hierarchy of uniform grids, levels 0..max_level (reference fem.py:300)."""
    return GridHierarchy(dim, max_level, degree, device)


def manufactured(dim):
    """The reference's benchmark solution u = prod sin(2 pi x_d) (1 + sin pi t) e^{-t/2}
    (reference fem.py:305-339); returns (u_exact, f_source, g_boundary)."""

    def spatial(x):
        x = np.atleast_2d(x)
        s = np.ones(x.shape[0])
        for d in range(dim):
            s = s * np.sin(2.0 * np.pi * x[:, d])
        return s

    def T(t):
        return (1.0 + np.sin(np.pi * t)) * np.exp(-0.5 * t)

    def dT(t):
        return np.exp(-0.5 * t) * (np.pi * np.cos(np.pi * t) - 0.5 * (1.0 + np.sin(np.pi * t)))

    def u_exact(x, t):
        return spatial(x) * T(t)

    def f_source(x, t):
        return spatial(x) * (dT(t) + 4.0 * np.pi ** 2 * dim * T(t))

    # the same functions in separable form (u = T(t) prod s(x_d), f = F(t) prod s(x_d)): device
    # load vectors, right-hand sides and L2 errors use it (load_vector_device, irk.StageSystem)
    sep = SeparableSolution(dim, s=lambda x: np.sin(2.0 * np.pi * np.asarray(x)), T=T,
                            F=lambda t: dT(t) + 4.0 * np.pi ** 2 * dim * T(t))
    u_exact.separable, f_source.separable = sep.field_view(sep.T), sep.field_view(sep.F)
    u_exact.solution = f_source.solution = sep
    return u_exact, f_source, u_exact


@dataclass
class SeparableSolution:
    """u(x,t) = T(t) prod_d s(x_d) with f = (T' + c_lap T) prod_d s: the configs' manufactured
    solution sin(pi x) sin(pi y) [sin(pi z)] e^{-t} (BASELINE.json configs) is the default."""

    dim: int
    s: callable = None
    T: callable = None
    F: callable = None  # time factor of the source

    def __post_init__(self):
        if self.s is None:
            d = self.dim
            self.s = lambda x: np.sin(np.pi * np.asarray(x))
            self.T = lambda t: np.exp(-t)
            self.F = lambda t: (d * np.pi ** 2 - 1.0) * np.exp(-t)

    def field_view(self, time_factor):
        """One separable field time_factor(t) prod s(x_d) (u: T, the source f: F) in the form the
        device quadratures read (.s and the time factor as both .T and .F)."""
        return SeparableSolution(self.dim, s=self.s, T=time_factor, F=time_factor)

    def callables(self):
        def spatial(x):
            x = np.atleast_2d(x)
            v = np.ones(x.shape[0])
            for d in range(self.dim):
                v = v * self.s(x[:, d])
            return v

        u = lambda x, t: spatial(x) * self.T(t)
        f = lambda x, t: spatial(x) * self.F(t)
        u.separable, f.separable = self.field_view(self.T), self.field_view(self.F)
        u.solution = f.solution = self
        return (u, f, u)


@dataclass
class HeatProblem:
    """Time-stepping setup on a hierarchy (reference fem.py:342-381)."""

    hierarchy: GridHierarchy
    tau: float
    t0: float = 0.0
    steps: int = 10
    callables: tuple = field(default=None, repr=False)

    def __post_init__(self):
        if self.tau <= 0.0:
            raise ConfigurationError("tau must be positive")
        if self.steps < 1:
            raise ConfigurationError("steps must be >= 1")
        if self.callables is None:
            self.callables = manufactured(self.hierarchy.dim)

    @property
    def u_exact(self):
        return self.callables[0]

    @property
    def f_source(self):
        return self.callables[1]

    def initial_condition(self):
        hier = self.hierarchy
        return self.u_exact(hier.node_coords(hier.max_level), self.t0)

    def load(self, t):
        hier = self.hierarchy
        return hier.load_vector(hier.max_level, self.f_source, t)

    def error(self, u, t):
        hier = self.hierarchy
        return hier.l2_error(hier.max_level, u, self.u_exact, t)
