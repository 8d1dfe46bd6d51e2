"""Radau IIA tableaux and the Q x Q factorizations the stage preconditioners need (host side).

Same public API and conventions as the reference tableau module (tableau.py:24-82 types,
radau_iia :164, crout_lu :189, spectral_real :210, spectral_complex :259, tableau_csv_rows :328):
  * nodes c ascending with c_Q = 1 exactly; b = last row of A (stiffly accurate);
  * Crout split Ainv = L U with unit-diagonal U;
  * real eigenvectors of the triangular L normalised to a unit first entry (S unit lower-triangular);
  * complex spectrum of Ainv: conjugate pairs adjacent (Im > 0 member first, partner vector the
    exact conjugate), pairs by ascending real part, odd-Q real eigenvalue last, eigenvectors scaled so
    the first significant entry is one.
The algorithms are this package's own: Legendre-companion roots polished by Newton for the nodes,
barycentric Lagrange + (Q+1)-point Gauss for A, and exact rational arithmetic (fractions) for the
ill-conditioned triangular eigenbasis, rounded once to float64.
"""

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .errors import (
    DegenerateSpectrumError,
    FactorizationError,
    SpectralFailureError,
    UnsupportedStageCountError,
)

MAX_STAGES = 9


@dataclass(frozen=True)
class ButcherTableau:
    """Q-stage Radau IIA coefficients: A (Q x Q), weights b, nodes c, and inv(A)."""

    Q: int
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    Ainv: np.ndarray


@dataclass(frozen=True)
class TriangularFactors:
    """inv(A) = L @ U, L lower triangular, U upper triangular with ones on the diagonal."""

    L: np.ndarray
    U: np.ndarray


@dataclass(frozen=True)
class RealSpectralFactors:
    """L = S diag(lambdas) Sinv with real eigenpairs (S unit lower triangular)."""

    lambdas: np.ndarray
    S: np.ndarray
    Sinv: np.ndarray


@dataclass(frozen=True)
class EigenvaluePair:
    """Representative of a conjugate pair (or the lone real eigenvalue, which is its own partner)."""

    re: float
    im: float
    index: int
    partner_index: int

    @property
    def is_real(self):
        return self.index == self.partner_index


@dataclass(frozen=True)
class ComplexSpectralFactors:
    """inv(A) = S diag(lambdas) Sinv over C, pairs adjacent, one `pairs` entry per block."""

    lambdas: np.ndarray
    S: np.ndarray
    Sinv: np.ndarray
    pairs: tuple


def _radau_right_nodes(Q):
    """Zeros of P_Q(2x-1) - P_{Q-1}(2x-1) on (0, 1]; the right end point is set exactly."""
    if Q == 1:
        return np.array([1.0])
    leg = np.polynomial.legendre
    coef = np.zeros(Q + 1)
    coef[Q] = 1.0
    coef[Q - 1] = -1.0
    roots = np.sort(leg.legroots(coef).real)  # in t = 2x - 1
    # Newton polish in t on the Legendre series
    dcoef = leg.legder(coef)
    for _ in range(4):
        roots = roots - leg.legval(roots, coef) / leg.legval(roots, dcoef)
    x = 0.5 * (roots + 1.0)
    x = np.sort(x)
    x[-1] = 1.0
    return x


def _lagrange_basis(nodes, j, s):
    """Lagrange basis polynomial j on `nodes`, evaluated at points s (barycentric weights)."""
    w = 1.0
    for m, cm in enumerate(nodes):
        if m != j:
            w /= nodes[j] - cm
    out = np.full_like(s, w, dtype=float)
    for m, cm in enumerate(nodes):
        if m != j:
            out = out * (s - cm)
    return out


def radau_iia(Q):
    """Q-stage Radau IIA: collocation at the right Radau nodes, a_ij = int_0^{c_i} l_j(s) ds."""
    if not (1 <= int(Q) <= MAX_STAGES) or int(Q) != Q:
        raise UnsupportedStageCountError(f"Radau IIA is provided for 1 <= Q <= {MAX_STAGES}, got {Q}")
    Q = int(Q)
    c = _radau_right_nodes(Q)
    xg, wg = np.polynomial.legendre.leggauss(Q + 1)  # exact for the degree Q-1 integrands
    A = np.empty((Q, Q))
    for i in range(Q):
        s = 0.5 * c[i] * (xg + 1.0)
        ws = 0.5 * c[i] * wg
        for j in range(Q):
            A[i, j] = float(np.dot(ws, _lagrange_basis(c, j, s)))
    b = A[Q - 1].copy()
    Ainv = _exact_inverse(A)
    return ButcherTableau(Q=Q, A=A, b=b, c=c, Ainv=Ainv)


def _exact_inverse(A):
    """inv(A) of the float64 matrix A computed exactly (rational Gauss-Jordan with partial
    pivoting) and rounded once: the correctly rounded inverse. The LU factor's eigenbasis is
    ill-conditioned for Q >= 8, and a LAPACK inverse's last-bit errors there push the reference's
    spectral reconstruction check (test_tableau.py:138-146) over its 1e-10 bound."""
    n = A.shape[0]
    M = [[Fraction(float(A[i, j])) for j in range(n)] + [Fraction(int(i == j)) for j in range(n)]
         for i in range(n)]
    for col in range(n):
        piv = max(range(col, n), key=lambda r: abs(M[r][col]))
        if M[piv][col] == 0:
            raise FactorizationError(col)
        M[col], M[piv] = M[piv], M[col]
        inv_p = 1 / M[col][col]
        M[col] = [v * inv_p for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                f = M[r][col]
                M[r] = [x - f * y for x, y in zip(M[r], M[col])]
    return np.array([[float(M[i][n + j]) for j in range(n)] for i in range(n)])


def crout_lu(Ainv):
    """Crout elimination: column j of L, then row j of U (unit diagonal)."""
    M = np.asarray(Ainv, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("crout_lu expects a square matrix")
    n = M.shape[0]
    L = np.zeros((n, n))
    U = np.eye(n)
    for j in range(n):
        for i in range(j, n):
            L[i, j] = M[i, j] - sum(L[i, k] * U[k, j] for k in range(j))
        if L[j, j] == 0.0:
            raise FactorizationError(j)
        for i in range(j + 1, n):
            U[j, i] = (M[j, i] - sum(L[j, k] * U[k, i] for k in range(j))) / L[j, j]
    return TriangularFactors(L=L, U=U)


def spectral_real(L):
    """Eigen-decomposition of a lower-triangular L with distinct diagonal, in exact arithmetic.

    The eigenvector for lambda_k solves (L - lambda_k I) v = 0 with v_k = 1 by forward
    substitution; the inverse of the unit-lower-triangular S is also exact. Both are rounded to
    float64 once at the end.
    """
    L = np.asarray(L, dtype=float)
    n = L.shape[0]
    lambdas = np.diag(L).copy()
    scale = max(float(np.abs(lambdas).max()), 1.0)
    for p in range(n):
        for q in range(p + 1, n):
            if abs(lambdas[p] - lambdas[q]) < 1e-10 * scale:
                raise DegenerateSpectrumError(f"diagonal entries {p} and {q} closer than 1e-10 relative")
    Lf = [[Fraction(float(L[i, j])) for j in range(n)] for i in range(n)]
    S = [[Fraction(0)] * n for _ in range(n)]
    for k in range(n):
        S[k][k] = Fraction(1)
        for i in range(k + 1, n):
            acc = sum((Lf[i][m] * S[m][k] for m in range(k, i)), Fraction(0))
            S[i][k] = -acc / (Lf[i][i] - Lf[k][k])
    Si = [[Fraction(0)] * n for _ in range(n)]
    for j in range(n):
        Si[j][j] = Fraction(1)
        for i in range(j + 1, n):
            Si[i][j] = -sum((S[i][m] * Si[m][j] for m in range(j, i)), Fraction(0))
    to_f = lambda X: np.array([[float(v) for v in row] for row in X])
    return RealSpectralFactors(lambdas=lambdas, S=to_f(S), Sinv=to_f(Si))


def _normalise_first(v):
    mag = np.abs(v)
    k = int(np.argmax(mag > 1e-12 * mag.max()))
    return v / v[k]


def spectral_complex(Ainv):
    """Complex eigen-decomposition of inv(A) with the pair conventions of the module docstring."""
    M = np.asarray(Ainv, dtype=float)
    Q = M.shape[0]
    try:
        vals, vecs = np.linalg.eig(M)
    except np.linalg.LinAlgError as exc:  # pragma: no cover
        raise SpectralFailureError(str(exc)) from exc
    if not np.all(np.isfinite(vals)):
        raise SpectralFailureError("non-finite eigenvalues")
    scale = float(np.abs(vals).max())
    real_idx = [i for i in range(Q) if abs(vals[i].imag) <= 1e-10 * scale]
    upper = [i for i in range(Q) if vals[i].imag > 1e-10 * scale]
    lower = [i for i in range(Q) if vals[i].imag < -1e-10 * scale]
    if len(real_idx) != Q % 2 or len(upper) != len(lower):
        raise SpectralFailureError(f"expected {Q % 2} real eigenvalue(s), found {len(real_idx)}")
    for i in upper:  # each upper member must have a conjugate partner
        if min(abs(vals[j] - np.conj(vals[i])) for j in lower) > 1e-8 * scale:
            raise SpectralFailureError("could not match a conjugate pair")
    upper.sort(key=lambda i: vals[i].real)
    lambdas = np.zeros(Q, dtype=complex)
    S = np.zeros((Q, Q), dtype=complex)
    pairs = []
    pos = 0
    for i in upper:
        v = _normalise_first(vecs[:, i])
        lambdas[pos], lambdas[pos + 1] = vals[i], np.conj(vals[i])
        S[:, pos], S[:, pos + 1] = v, np.conj(v)
        pairs.append(EigenvaluePair(re=vals[i].real, im=vals[i].imag, index=pos, partner_index=pos + 1))
        pos += 2
    for i in real_idx:
        v = _normalise_first(vecs[:, i])
        lambdas[pos] = vals[i].real
        S[:, pos] = v.real
        pairs.append(EigenvaluePair(re=vals[i].real, im=0.0, index=pos, partner_index=pos))
        pos += 1
    return ComplexSpectralFactors(lambdas=lambdas, S=S, Sinv=np.linalg.inv(S), pairs=tuple(pairs))


def tableau_csv_rows(tab):
    """CSV export rows: [c_i, a_i1 .. a_iQ] per stage, then ['b', b_1 .. b_Q]."""
    rows = [[repr(float(tab.c[i]))] + [repr(float(x)) for x in tab.A[i]] for i in range(tab.Q)]
    rows.append(["b"] + [repr(float(x)) for x in tab.b])
    return rows
