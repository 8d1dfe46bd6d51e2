/* Oracle fast path (TEST ONLY): a banded matrix applied along one tensor axis.
 *
 * Same operation as the reference's dense contraction (fem.py:37-41, `_contract`: moveaxis ->
 * reshape -> (n x n) @ (n x rest) -> moveaxis) restricted to the matrix's nonzero band, which for
 * the assembled 1D Q_k mass / stiffness matrices (fem.py:21-34 generalised), the Q_k prolongation
 * (fem.py:287-297) and its transpose is at most 2k+1 wide. The array is viewed as (A, n_in, B)
 * around the contracted axis; out[a, i, b] = sum_{j < bw} vals[i][j] * in[a, col0[i] + j, b].
 * Products are summed in column order, so results agree with the dense BLAS contraction to
 * rounding (checked in tests/test_oracle_fast.py). OpenMP over (a, i).
 */
#include <stddef.h>

void band_axis(const double* in, double* out, long long A, int nin, int nout, long long B,
               const int* col0, const double* vals, int bw, int acc) {
  (void)nin;
#pragma omp parallel for collapse(2) schedule(static)
  for (long long a = 0; a < A; ++a) {
    for (int i = 0; i < nout; ++i) {
      double* o = out + ((size_t)a * nout + i) * B;
      const double* v = vals + (size_t)i * bw;
      const double* base = in + ((size_t)a * nin + col0[i]) * B;
      if (B == 1) {
        double s = 0.0;
        for (int j = 0; j < bw; ++j) s += v[j] * base[j];
        o[0] = acc ? o[0] + s : s;
      } else {
        const double c0 = v[0];
        if (acc)
          for (long long b = 0; b < B; ++b) o[b] += c0 * base[b];
        else
          for (long long b = 0; b < B; ++b) o[b] = c0 * base[b];
        for (int j = 1; j < bw; ++j) {
          const double c = v[j];
          if (c == 0.0) continue;
          const double* src = base + (size_t)j * B;
          for (long long b = 0; b < B; ++b) o[b] += c * src[b];
        }
      }
    }
  }
}

/* y = a*x + b*y style helpers are left to numpy; this file holds only the contraction. */
