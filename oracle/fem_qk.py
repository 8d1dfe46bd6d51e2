"""Oracle: the reference's Kronecker-form FEM discretisation generalised to Q_k (TEST ONLY).

Restates reference fem.py with the element degree k as a parameter:
  * dense assembled 1D matrices per level (fem.py:21-34 for k=1; here (k+1)x(k+1) element tables
    from the exact (k+1)-point Gauss rule on Gauss-Lobatto-Legendre nodes);
  * one dense contraction per tensor axis, moveaxis -> matmul -> moveaxis (fem.py:37-41);
  * M = M1 x M1 x M1, K = sum of Kronecker terms (fem.py:120-143), shifted/constrained forms
    (fem.py:145-170), Kronecker diagonal with 1.0 on boundary rows (fem.py:172-187);
  * Q_k embedding prolongation and its transpose (fem.py:189-211, _prolongation_1d :287-297);
  * load vector and L2 error with the (k+1)-point Gauss rule (fem.py:220-273).
At k = 1 this is the reference algorithm and reproduces it (tests/test_oracle_golden.py).
"""

import numpy as np


def gll_nodes01(k):
    """Gauss-Lobatto-Legendre nodes on [0, 1]: end points and the roots of P_k'."""
    if k == 1:
        return np.array([0.0, 1.0])
    inner = np.polynomial.legendre.Legendre.basis(k).deriv().roots()
    x = np.concatenate(([-1.0], np.sort(inner.real), [1.0]))
    x = 0.5 * (x + 1.0)
    x[0], x[-1] = 0.0, 1.0
    if k % 2 == 0:
        x[k // 2] = 0.5
    # enforce the exact reflection symmetry of the node set
    for i in range(k // 2):
        x[k - i] = 1.0 - x[i]
    return x


def gauss01(m):
    x, w = np.polynomial.legendre.leggauss(m)
    return 0.5 * (x + 1.0), 0.5 * w


def lagrange_values(nodes, a, x):
    x = np.asarray(x, dtype=float)
    v = np.ones_like(x)
    for m, xm in enumerate(nodes):
        if m != a:
            v = v * (x - xm) / (nodes[a] - xm)
    return v


def lagrange_derivs(nodes, a, x):
    x = np.asarray(x, dtype=float)
    tot = np.zeros_like(x)
    for m, xm in enumerate(nodes):
        if m == a:
            continue
        t = np.full_like(x, 1.0 / (nodes[a] - xm))
        for l, xl in enumerate(nodes):
            if l != a and l != m:
                t = t * (x - xl) / (nodes[a] - xl)
        tot = tot + t
    return tot


def reference_element(k):
    """(M_hat, K_hat) on [0,1] with the exact (k+1)-point Gauss rule."""
    nodes = gll_nodes01(k)
    xg, wg = gauss01(k + 1)
    phi = np.stack([lagrange_values(nodes, a, xg) for a in range(k + 1)])
    dphi = np.stack([lagrange_derivs(nodes, a, xg) for a in range(k + 1)])
    Mh = (phi * wg) @ phi.T
    Kh = (dphi * wg) @ dphi.T
    return 0.5 * (Mh + Mh.T), 0.5 * (Kh + Kh.T)


def assemble_1d(elem, n_elems, k):
    n = k * n_elems + 1
    out = np.zeros((n, n))
    for e in range(n_elems):
        out[k * e : k * e + k + 1, k * e : k * e + k + 1] += elem
    return out


FAST = False  # banded fast path (oracle/fastband.c); the dense form below is the reference's
FAST_MIN = 1 << 17  # smaller arrays keep the dense numpy contraction (no OpenMP fork per call)
FAST_MIN_AXIS = 129  # the dense contraction costs n_ax per entry: the band only pays on long axes


def contract(mat, arr, axis):
    """Dense matrix along one tensor axis (reference fem.py:37-41). With FAST (or
    Hierarchy(fast=True)) the same product over the matrix's nonzero band only."""
    if FAST and mat.shape[1] >= FAST_MIN_AXIS and np.size(arr) >= FAST_MIN:
        from .fastband import band_contract
        return band_contract(mat, arr, axis)
    moved = np.moveaxis(arr, axis, 0)
    res = mat @ moved.reshape(moved.shape[0], -1)
    return np.moveaxis(res.reshape((mat.shape[0],) + moved.shape[1:]), 0, axis)


def prolongation_1d(k, n_coarse_elems):
    """Dense Q_k embedding: fine node values of the coarse interpolant."""
    nodes = gll_nodes01(k)
    nc = k * n_coarse_elems + 1
    nf = 2 * k * n_coarse_elems + 1
    P = np.zeros((nf, nc))
    for i in range(nf):
        ec = min(i // (2 * k), n_coarse_elems - 1)
        f = i - 2 * k * ec
        pos = 0.5 * nodes[f] if f <= k else 0.5 + 0.5 * nodes[f - k]
        for j in range(k + 1):
            P[i, k * ec + j] = lagrange_values(nodes, j, pos)
    P[np.abs(P) < 1e-15] = 0.0
    # rows at coarse nodes are exact unit rows
    for i in range(nf):
        ec = min(i // (2 * k), n_coarse_elems - 1)
        f = i - 2 * k * ec
        if f == 0 or f == 2 * k or (k % 2 == 0 and f == k):
            j = 0 if f == 0 else (k if f == 2 * k else k // 2)
            P[i, :] = 0.0
            P[i, k * ec + j] = 1.0
    return P


class Level:
    def __init__(self, index, dim, k):
        self.index, self.dim, self.k = index, dim, k
        self.n_elems = 2 ** index
        self.n_per_axis = k * self.n_elems + 1
        self.h = 1.0 / self.n_elems
        Mh, Kh = reference_element(k)
        self.elem_mass = self.h * Mh
        self.elem_stiffness = Kh / self.h
        self.mass_1d = assemble_1d(self.elem_mass, self.n_elems, k)
        self.stiffness_1d = assemble_1d(self.elem_stiffness, self.n_elems, k)
        nodes = gll_nodes01(k)
        coords = np.concatenate([(e + nodes[:-1]) * self.h for e in range(self.n_elems)] + [[1.0]])
        self.coords = coords
        inter = np.ones(self.n_per_axis, dtype=bool)
        inter[0] = inter[-1] = False
        mask = inter
        for _ in range(dim - 1):
            mask = np.logical_and.outer(mask, inter)
        self.interior_mask = mask.ravel()

    @property
    def shape(self):
        return (self.n_per_axis,) * self.dim

    @property
    def n_dofs(self):
        return self.n_per_axis ** self.dim


class Hierarchy:
    """Oracle GridHierarchy(dim, max_level, k)."""

    def __init__(self, dim, max_level, k=1, fast=False):
        self.dim, self.max_level, self.k = dim, max_level, k
        self.levels = [Level(l, dim, k) for l in range(max_level + 1)]
        if fast:  # process-wide switch: every contraction of the oracle takes the banded path
            global FAST
            FAST = True

    @property
    def finest(self):
        return self.levels[-1]

    @property
    def n(self):
        return self.finest.n_dofs

    def _kron_apply(self, level, u, factors):
        lvl = self.levels[level]
        lead = u.shape[:-1]
        w = np.asarray(u, dtype=float).reshape(lead + lvl.shape)
        off = len(lead)
        for ax, mat in enumerate(factors):
            w = contract(mat, w, off + ax)
        return w.reshape(lead + (lvl.n_dofs,))

    def _mass_stiff_fast(self, level, u):
        """(M u, K u) by sum factorisation over banded 1D factors (fast path only): the same
        Kronecker products as apply_mass / apply_stiffness with shared partial sweeps."""
        from .fastband import band_contract as bc
        lvl = self.levels[level]
        lead = u.shape[:-1]
        off = len(lead)
        w = np.asarray(u, dtype=float).reshape(lead + lvl.shape)
        Mm, Kk = lvl.mass_1d, lvl.stiffness_1d
        m, k = bc(Mm, w, off + self.dim - 1), bc(Kk, w, off + self.dim - 1)   # last axis
        for ax in range(self.dim - 2, -1, -1):
            m, k = bc(Mm, m, off + ax), bc(Mm, k, off + ax, out=bc(Kk, m, off + ax))
        return m.reshape(lead + (lvl.n_dofs,)), k.reshape(lead + (lvl.n_dofs,))

    def apply_mass(self, level, u):
        lvl = self.levels[level]
        return self._kron_apply(level, u, [lvl.mass_1d] * self.dim)

    def apply_stiffness(self, level, u):
        lvl = self.levels[level]
        if FAST and self.levels[level].n_per_axis >= FAST_MIN_AXIS:
            return self._mass_stiff_fast(level, u)[1]
        out = 0.0
        for d in range(self.dim):
            facs = [lvl.stiffness_1d if ax == d else lvl.mass_1d for ax in range(self.dim)]
            out = out + self._kron_apply(level, u, facs)
        return out

    def apply_shifted(self, level, lam, tau, u):
        if FAST and self.levels[level].n_per_axis >= FAST_MIN_AXIS:
            mu, ku = self._mass_stiff_fast(level, u)
        else:
            mu = self.apply_mass(level, u)
            ku = self.apply_stiffness(level, u)
        if np.ndim(lam) == 0:
            return lam * mu + tau * ku
        return np.asarray(lam).reshape((-1,) + (1,) * (np.ndim(u) - 1)) * mu + tau * ku

    def apply_constrained(self, level, lam, tau, u):
        mask = self.levels[level].interior_mask
        v = self.apply_shifted(level, lam, tau, np.where(mask, u, 0.0))
        return np.where(mask, v, u)

    def apply_stage(self, level, DM, DK, u, constrained=False):
        """(D_M (x) M + D_K (x) K) u on (Q, n) stage vectors (SPEC irk:A operator form)."""
        mask = self.levels[level].interior_mask
        ui = np.where(mask, u, 0.0) if constrained else u
        if FAST and self.levels[level].n_per_axis >= FAST_MIN_AXIS:
            mu, ku = self._mass_stiff_fast(level, ui)
        else:
            mu = self.apply_mass(level, ui)
            ku = self.apply_stiffness(level, ui)
        v = np.asarray(DM) @ mu + np.asarray(DK) @ ku
        return np.where(mask, v, u) if constrained else v

    def constrain(self, level, vec, boundary_values=0.0):
        out = np.array(vec, copy=True, dtype=float)
        out[..., ~self.levels[level].interior_mask] = boundary_values
        return out

    def operator_diagonal(self, level, lam, tau):
        lvl = self.levels[level]
        dm1, dk1 = np.diag(lvl.mass_1d), np.diag(lvl.stiffness_1d)
        dm = dm1
        for _ in range(self.dim - 1):
            dm = np.multiply.outer(dm, dm1)
        dk = np.zeros(lvl.shape)
        for d in range(self.dim):
            term = np.ones(())
            for ax in range(self.dim):
                term = np.multiply.outer(term, dk1 if ax == d else dm1)
            dk = dk + term
        return np.where(lvl.interior_mask, (lam * dm + tau * dk).ravel(), 1.0)

    def prolong(self, coarse_level, uc):
        P = prolongation_1d(self.k, self.levels[coarse_level].n_elems)
        lead = uc.shape[:-1]
        w = np.asarray(uc, dtype=float).reshape(lead + self.levels[coarse_level].shape)
        for ax in range(self.dim):
            w = contract(P, w, len(lead) + ax)
        return w.reshape(lead + (-1,))

    def restrict(self, fine_level, rf):
        P = prolongation_1d(self.k, self.levels[fine_level - 1].n_elems)
        lead = rf.shape[:-1]
        w = np.asarray(rf, dtype=float).reshape(lead + self.levels[fine_level].shape)
        for ax in range(self.dim):
            w = contract(P.T, w, len(lead) + ax)
        return w.reshape(lead + (-1,))

    def node_coords(self, level):
        c = self.levels[level].coords
        mesh = np.meshgrid(*([c] * self.dim), indexing="ij")
        return np.stack([m.ravel() for m in mesh], axis=-1)

    def _gauss_1d(self, level):
        lvl = self.levels[level]
        k = self.k
        xg, wg = gauss01(k + 1)
        nodes = gll_nodes01(k)
        pts = ((np.arange(lvl.n_elems)[:, None] + xg[None, :]) * lvl.h).ravel()
        shape = np.stack([lagrange_values(nodes, a, xg) for a in range(k + 1)])
        return pts, wg, shape

    def load_vector(self, level, f, t):
        lvl = self.levels[level]
        k = self.k
        pts1, wg, shape = self._gauss_1d(level)
        mesh = np.meshgrid(*([pts1] * self.dim), indexing="ij")
        pts = np.stack([m.ravel() for m in mesh], axis=-1)
        vals = np.asarray(f(pts, t), dtype=float).reshape((pts1.size,) * self.dim)
        B = np.zeros((lvl.n_per_axis, pts1.size))
        for e in range(lvl.n_elems):
            for a in range(k + 1):
                B[k * e + a, (k + 1) * e : (k + 1) * (e + 1)] += shape[a] * wg * lvl.h
        for ax in range(self.dim):
            vals = contract(B, vals, ax)
        return vals.ravel()

    def l2_error(self, level, u_nodal, u_exact, t):
        lvl = self.levels[level]
        k = self.k
        pts1, wg, shape = self._gauss_1d(level)
        I = np.zeros((pts1.size, lvl.n_per_axis))
        for e in range(lvl.n_elems):
            for a in range(k + 1):
                I[(k + 1) * e : (k + 1) * (e + 1), k * e + a] = shape[a]
        w = np.asarray(u_nodal, dtype=float).reshape(lvl.shape)
        for ax in range(self.dim):
            w = contract(I, w, ax)
        mesh = np.meshgrid(*([pts1] * self.dim), indexing="ij")
        pts = np.stack([m.ravel() for m in mesh], axis=-1)
        diff = w.ravel() - u_exact(pts, t)
        w1 = np.tile(wg * lvl.h, lvl.n_elems)
        wt = np.ones(())
        for _ in range(self.dim):
            wt = np.multiply.outer(wt, w1)
        return float(np.sqrt(np.sum(wt.ravel() * diff ** 2)))
