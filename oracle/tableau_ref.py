"""Oracle: Radau IIA tableau and Q x Q factorizations, restated from reference tableau.py (TEST ONLY).

radau_iia (tableau.py:164-186): right-Radau nodes as roots of d^{Q-1}/dx^{Q-1}[x^{Q-1}(x-1)^Q] found by
a 2e5-point sign scan + bisection (:112-148), a_ij by the Q-point Gauss rule on [0, c_i] (:174-183),
b = last row of A, Ainv = inv(A). crout_lu (:189-207). spectral_real in extended precision (:210-249).
spectral_complex with adjacent conjugate pairs and the odd-Q real eigenvalue last (:259-325).
"""

from math import comb

import numpy as np


def _radau_poly(Q):
    base = np.zeros(2 * Q)
    for k in range(Q + 1):
        base[Q - 1 + k] = comb(Q, k) * (-1) ** (Q - k)
    order = Q - 1
    out = np.zeros(2 * Q - order)
    for m in range(order, 2 * Q):
        if base[m] != 0.0:
            f = 1.0
            for j in range(m, m - order, -1):
                f *= j
            out[m - order] = base[m] * f
    return out


def _horner(c, x):
    y = 0.0
    for a in c[::-1]:
        y = y * x + a
    return y


def radau_nodes(Q):
    if Q == 1:
        return np.array([1.0])
    c = _radau_poly(Q)
    xs = np.linspace(0.0, 1.0, 200001)
    vals = (xs[:, None] ** np.arange(len(c))[None, :]) @ c
    roots = []
    for i in range(len(xs) - 1):
        fa, fb = vals[i], vals[i + 1]
        if fa == 0.0 and 0.0 < xs[i] < 1.0 - 1e-9:
            roots.append(xs[i])
            continue
        if fa * fb < 0.0:
            lo, hi, flo = xs[i], xs[i + 1], fa
            while hi - lo > 1e-17:
                mid = 0.5 * (lo + hi)
                if mid in (lo, hi):
                    break
                fm = _horner(c, mid)
                if fm == 0.0:
                    lo = hi = mid
                elif flo * fm < 0.0:
                    hi = mid
                else:
                    lo, flo = mid, fm
            roots.append(0.5 * (lo + hi))
    roots = sorted(r for r in roots if r < 1.0 - 1e-9)
    return np.array(roots + [1.0])


def radau_iia(Q):
    c = radau_nodes(Q)
    xg, wg = np.polynomial.legendre.leggauss(Q)
    A = np.zeros((Q, Q))
    for i in range(Q):
        pts = 0.5 * c[i] * (xg + 1.0)
        w = 0.5 * c[i] * wg
        for j in range(Q):
            num = np.ones_like(pts)
            den = 1.0
            for m in range(Q):
                if m != j:
                    num = num * (pts - c[m])
                    den *= c[j] - c[m]
            A[i, j] = np.sum(w * (num / den))
    return dict(Q=Q, A=A, b=A[-1].copy(), c=c, Ainv=np.linalg.inv(A))


def crout_lu(M):
    n = M.shape[0]
    L, U = np.zeros((n, n)), np.eye(n)
    for j in range(n):
        for i in range(j, n):
            L[i, j] = M[i, j] - L[i, :j] @ U[:j, j]
        for i in range(j + 1, n):
            U[j, i] = (M[j, i] - L[j, :j] @ U[:j, i]) / L[j, j]
    return L, U


def spectral_real(L):
    n = L.shape[0]
    lam = np.diag(L).copy()
    Lx = L.astype(np.longdouble)
    S = np.zeros((n, n), dtype=np.longdouble)
    for k in range(n):
        v = np.zeros(n, dtype=np.longdouble)
        v[k] = 1.0
        for i in range(k + 1, n):
            v[i] = -(Lx[i, k:i] @ v[k:i]) / (Lx[i, i] - Lx[k, k])
        S[:, k] = v
    Si = np.zeros((n, n), dtype=np.longdouble)
    for j in range(n):
        x = np.zeros(n, dtype=np.longdouble)
        x[j] = 1.0
        for i in range(j + 1, n):
            x[i] = -(S[i, :i] @ x[:i])
        Si[:, j] = x
    return lam, S.astype(float), Si.astype(float)


def spectral_complex(Ainv):
    """Returns (lambdas, S, Sinv, pairs) with pairs = [(re, im, index, partner_index), ...]."""
    Q = Ainv.shape[0]
    vals, vecs = np.linalg.eig(Ainv)
    order = np.argsort(-vals.imag, kind="stable")
    remaining = list(order)
    scale = np.abs(vals).max()
    groups, reals = [], []
    while remaining:
        i = remaining.pop(0)
        if abs(vals[i].imag) <= 1e-10 * scale:
            reals.append(i)
            continue
        j = min(remaining, key=lambda jj: abs(vals[jj] - np.conj(vals[i])))
        remaining.remove(j)
        rep = i if vals[i].imag > 0 else j
        groups.append((vals[rep], vecs[:, rep]))
    groups.sort(key=lambda g: g[0].real)

    def first_one(v):
        mag = np.abs(v)
        return v / v[int(np.argmax(mag > 1e-12 * mag.max()))]

    lam = np.zeros(Q, dtype=complex)
    S = np.zeros((Q, Q), dtype=complex)
    pairs, pos = [], 0
    for l, v in groups:
        v = first_one(v)
        lam[pos], lam[pos + 1] = l, np.conj(l)
        S[:, pos], S[:, pos + 1] = v, np.conj(v)
        pairs.append((l.real, l.imag, pos, pos + 1))
        pos += 2
    for i in reals:
        v = first_one(vecs[:, i])
        lam[pos] = vals[i].real
        S[:, pos] = v.real
        pairs.append((vals[i].real, 0.0, pos, pos))
        pos += 1
    return lam, S, np.linalg.inv(S), pairs
