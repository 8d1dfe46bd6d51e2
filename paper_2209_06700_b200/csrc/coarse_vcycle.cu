// Fused V-cycle on the coarsest levels of a whole-mesh 2D or 3D hierarchy (block family, direct
// coarse solve), sm_100a, fp64. A 2D level is a 3D one with a single x plane (degenerate x axis: the
// x factors of M and K are 1 and 0, the x sweeps of the operator and the transfers vanish).
//
// Below a few thousand nodes per block every kernel of the V-cycle (multigrid.py:110-140: Chebyshev
// steps, residual, restriction, prolongation, the coarse solve) is a launch of a few microseconds
// of latency: a level costs ~13 launches. Here levels 0..lc of one block run inside ONE CTA (the
// vectors of the levels below lc and the operator's sweep buffers in shared memory, level lc's
// vectors in global memory / L2): the same sequence of operations (multigrid._DeviceVCycle._cycle /
// _smooth / ChebyshevSmoother.apply, reference multigrid.py:65-140) with the operator applied by sum
// factorisation over the assembled 1D band rows, the transfers as three in-smem sweeps
// (vecops.cu transfer_value arithmetic) and the coarse level as the dense inverse (multigrid.py:
// 179-186). One CTA per block; the CTA's barriers separate the phases.
#include <cstdint>

#include "spk_internal.cuh"
#include "spk_vecops.cuh"
#include "stage_apply.cuh"

namespace {

#ifndef SPK_CV_NT
#define SPK_CV_NT 512
#endif
constexpr int CV_NT = SPK_CV_NT;

template <int K>
struct CVLevel {
  int m, mx, n;  // nodes per axis (y, z), nodes along x (1 in 2D), nodes
  __device__ CVLevel(int l, int dim)
      : m((K << l) + 1), mx(dim == 3 ? (K << l) + 1 : 1), n(mx * ((K << l) + 1) * ((K << l) + 1)) {}
};

// boundary node; mx == 1: degenerate x axis (2D), no x boundary
__device__ __forceinline__ bool cv_bnd(int x, int y, int z, int m, int mx) {
  return (mx > 1 && (x == 0 || x == m - 1)) || y == 0 || y == m - 1 || z == 0 || z == m - 1;
}

// band-row class of node i on an axis of m nodes (Band<K>::cls with the whole-axis convention)
template <int K>
__device__ __forceinline__ int cv_cls(int i, int m) {
  const int r = i % K;
  if (r != 0) return r;
  return i == 0 ? K : (i == m - 1 ? K + 1 : 0);
}

// Jacobi inverse diagonal of the constrained block operator at (x, y, z): 1 on boundary rows,
// else 1 / (lam' dm + tau' dk) with the Kronecker diagonal pieces (fem.py:172-187 association order)
template <int K>
__device__ __forceinline__ double cv_dinv(int x, int y, int z, int m, int nx, double lamp, double taup) {
  if (cv_bnd(x, y, z, m, nx)) return 1.0;
  const int E = (m - 1) / K, Ex = nx > 1 ? E : 0;
  double mx, kx, my, ky, mz, kz;
  class_diag1<K>(axis_class<K>(x, nx, Ex), Ex, mx, kx);
  class_diag1<K>(axis_class<K>(y, m, E), E, my, ky);
  class_diag1<K>(axis_class<K>(z, m, E), E, mz, kz);
  const double dm = (mx * my) * mz;
  const double dk = ((kx * my) * mz + (mx * ky) * mz) + (mx * my) * kz;
  return 1.0 / (lamp * dm + taup * dk);
}

struct CVShared {
  int dim;
  double* X[SPK_CV_LMAX + 1];
  double* B[SPK_CV_LMAX + 1];
  double* DI[SPK_CV_LMAX + 1];  // Jacobi inverse diagonal per level (computed once per launch)
  const int* CO[SPK_CV_LMAX + 1];  // packed node coordinates x | y << 10 | z << 20 per level (no div/mod)
  double *R, *D, *W, *T0, *T1, *T2, *T3;
  const double* bm;  // assembled band rows [K+2][2K+1] (reference element, h = 1)
  const double* bk;
};

// (A u)_i handed to epi(i, value) in the operator's last sweep (constrained: boundary entries of u
// read as 0, boundary rows = identity). The caller's per-node update rides on that sweep instead of
// taking a pass and a barrier of its own; it may overwrite u (read in the first sweep only).
template <int K, class Epi>
__device__ void cv_apply(const CVShared& S, int l, const double* u, double lamp, double taup, Epi&& epi) {
  constexpr int W = 2 * K + 1;
  const CVLevel<K> L(l, S.dim);
  const int m = L.m, n = L.n, mm = m * m, mx = L.mx;
  const int* co = S.CO[l];
  for (int i = threadIdx.x; i < n; i += CV_NT) {  // z: T0 = Mz u, T1 = Kz u
    const int cw = co[i], x = cw & 1023, y = (cw >> 10) & 1023, z = cw >> 20;
    const int c = cv_cls<K>(z, m);
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int d = 0; d < W; ++d) {
      const int zz = z + d - K;
      if (zz < 0 || zz >= m) continue;
      const double uv = cv_bnd(x, y, zz, m, mx) ? 0.0 : u[i + d - K];
      a = fma(S.bm[c * W + d], uv, a);
      b = fma(S.bk[c * W + d], uv, b);
    }
    S.T0[i] = a;
    S.T1[i] = b;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += CV_NT) {  // y: ma = My a, c = Ky a + My b -> p, q
    const int y = (co[i] >> 10) & 1023;
    const int c = cv_cls<K>(y, m);
    double ma = 0.0, cc = 0.0;
#pragma unroll
    for (int d = 0; d < W; ++d) {
      const int yy = y + d - K;
      if (yy < 0 || yy >= m) continue;
      const int j = i + (d - K) * m;
      ma = fma(S.bm[c * W + d], S.T0[j], ma);
      cc = fma(S.bk[c * W + d], S.T0[j], cc);
      cc = fma(S.bm[c * W + d], S.T1[j], cc);
    }
    if (mx == 1) {  // 2D: v = p (degenerate x factors Mx = 1, Kx = 0); boundary rows identity
      const int z = co[i] >> 20;
      epi(i, cv_bnd(0, y, z, m, 1) ? u[i] : fma(lamp, ma, taup * cc));
      continue;
    }
    S.T2[i] = fma(lamp, ma, taup * cc);  // p
    S.T3[i] = taup * ma;                 // q
  }
  __syncthreads();
  if (mx == 1) return;
  for (int i = threadIdx.x; i < n; i += CV_NT) {  // x: v = Mx p + Kx q ; boundary rows identity
    const int cw = co[i], x = cw & 1023, y = (cw >> 10) & 1023, z = cw >> 20;
    if (cv_bnd(x, y, z, m, mx)) {
      epi(i, u[i]);
      continue;
    }
    const int c = cv_cls<K>(x, m);
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < W; ++d) {
      const int xx = x + d - K;
      if (xx < 0 || xx >= m) continue;
      const int j = i + (d - K) * mm;
      acc = fma(S.bm[c * W + d], S.T2[j], acc);
      acc = fma(S.bk[c * W + d], S.T3[j], acc);
    }
    epi(i, acc);
  }
  __syncthreads();
}

// 1D transfer value (vecops.cu transfer_value): output node i along an axis, src[g * stride] is the
// input at global node g of that axis; Nc coarse elements
template <int K>
__device__ __forceinline__ double cv_tv(const double* P, int prolong, int Nc, int i, const double* src, int stride) {
  constexpr int PS = SPK_KMAX + 1;
  double val = 0.0;
  if (prolong) {
    const int ec = min(i / (2 * K), Nc - 1);
    const int f = i - 2 * K * ec;
#pragma unroll
    for (int j = 0; j <= K; ++j) val = fma(P[f * PS + j], src[(K * ec + j) * stride], val);
  } else {
    const int ec = i / K, r = i - ec * K;
    if (r != 0) {
#pragma unroll
      for (int f = 1; f < 2 * K; ++f) val = fma(P[f * PS + r], src[(2 * K * ec + f) * stride], val);
    } else {
      val = src[(2 * K * ec) * stride];
      if (ec < Nc) {
#pragma unroll
        for (int f = 1; f < 2 * K; ++f) val = fma(P[f * PS + 0], src[(2 * K * ec + f) * stride], val);
      }
      if (ec > 0) {
#pragma unroll
        for (int f = 1; f < 2 * K; ++f) val = fma(P[f * PS + K], src[(2 * K * (ec - 1) + f) * stride], val);
      }
    }
  }
  return val;
}

// B_{l-1} = mask(P^T R) (restriction of level l's residual), sweeps z, y, x
template <int K>
__device__ void cv_restrict(const CVShared& S, const double* P, int l) {
  const int mf = (K << l) + 1, mc = (K << (l - 1)) + 1, Nc = 1 << (l - 1);
  const int mxf = S.dim == 3 ? mf : 1;
  for (int i = threadIdx.x; i < mxf * mf * mc; i += CV_NT) {  // [xf][yf][zc]
    const int zc = i % mc, t = i / mc;
    S.T0[i] = cv_tv<K>(P, 0, Nc, zc, S.R + t * mf, 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < mxf * mc * mc; i += CV_NT) {  // [xf][yc][zc]
    const int zc = i % mc, t = i / mc, yc = t % mc, xf = t / mc;
    S.T1[i] = cv_tv<K>(P, 0, Nc, yc, S.T0 + xf * mf * mc + zc, mc);
  }
  __syncthreads();
  double* Bc = S.B[l - 1];
  if (S.dim == 2) {  // no x sweep: mask the (yc, zc) result
    for (int i = threadIdx.x; i < mc * mc; i += CV_NT) {
      const int zc = i % mc, yc = i / mc;
      Bc[i] = cv_bnd(0, yc, zc, mc, 1) ? 0.0 : S.T1[i];
    }
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < mc * mc * mc; i += CV_NT) {  // [xc][yc][zc], masked
    const int zc = i % mc, t = i / mc, yc = t % mc, xc = t / mc;
    const double val = cv_tv<K>(P, 0, Nc, xc, S.T1 + yc * mc + zc, mc * mc);
    Bc[i] = cv_bnd(xc, yc, zc, mc, mc) ? 0.0 : val;
  }
  __syncthreads();
}

// X_l += P X_{l-1}, sweeps z, y, x
template <int K>
__device__ void cv_prolong(const CVShared& S, const double* P, int l) {
  const int mf = (K << l) + 1, mc = (K << (l - 1)) + 1, Nc = 1 << (l - 1);
  const int mxc = S.dim == 3 ? mc : 1;
  const double* Xc = S.X[l - 1];
  for (int i = threadIdx.x; i < mxc * mc * mf; i += CV_NT) {  // [xc][yc][zf]
    const int zf = i % mf, t = i / mf;
    S.T0[i] = cv_tv<K>(P, 1, Nc, zf, Xc + t * mc, 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < mxc * mf * mf; i += CV_NT) {  // [xc][yf][zf]
    const int zf = i % mf, t = i / mf, yf = t % mf, xc = t / mf;
    S.T1[i] = cv_tv<K>(P, 1, Nc, yf, S.T0 + xc * mc * mf + zf, mf);
  }
  __syncthreads();
  double* Xf = S.X[l];
  if (S.dim == 2) {  // no x sweep
    for (int i = threadIdx.x; i < mf * mf; i += CV_NT) Xf[i] += S.T1[i];
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < mf * mf * mf; i += CV_NT) {  // [xf][yf][zf]
    const int zf = i % mf, t = i / mf, yf = t % mf, xf = t / mf;
    Xf[i] += cv_tv<K>(P, 1, Nc, xf, S.T1 + yf * mf + zf, mf * mf);
  }
  __syncthreads();
}

// Chebyshev smoothing at level l (ChebyshevSmoother.apply; zero start: r = b, x = 0)
template <int K>
__device__ void cv_smooth(const CVShared& S, const SpkCoarseArgs& a, int l, int blk, bool zero_start,
                          double lamp, double taup, bool& bad) {
  const CVLevel<K> L(l, S.dim);
  const int m = L.m, n = L.n;
  const int ncoef = 1 + 2 * (a.deg - 1);
  const double* cf = a.coef + ((long long)l * a.nblk + blk) * ncoef;
  const double theta = cf[0];
  double* X = S.X[l];
  const double* Bv = S.B[l];
  const double* DI = S.DI[l];
  if (!zero_start) {  // r = b - A x, d = Dinv r / theta (fused into the operator's last sweep)
    cv_apply<K>(S, l, X, lamp, taup, [&](int i, double w) {
      const double r = Bv[i] - w;
      S.R[i] = r;
      S.D[i] = (DI[i] * r) / theta;
    });
  } else {
    for (int i = threadIdx.x; i < n; i += CV_NT) {
      const double r = Bv[i];
      X[i] = 0.0;
      S.R[i] = r;
      S.D[i] = (DI[i] * r) / theta;
    }
    __syncthreads();
  }
  if (a.deg == 1) {
    for (int i = threadIdx.x; i < n; i += CV_NT) {
      const double xn = X[i] + S.D[i];
      X[i] = xn;
      bad |= !isfinite(xn);
    }
    __syncthreads();
    return;
  }
  for (int k = 0; k < a.deg - 1; ++k) {
    const double c1 = cf[1 + 2 * k], c2 = cf[2 + 2 * k];
    const bool last = (k == a.deg - 2);
    // w = A d with the step x += d; r -= w; d = c1 d + c2 Dinv r on each node in the same sweep
    cv_apply<K>(S, l, S.D, lamp, taup, [&](int i, double w) {
      const double d = S.D[i];
      const double xn = X[i] + d;
      const double r = S.R[i] - w;
      const double dn = c1 * d + c2 * (DI[i] * r);
      if (last) {
        const double xf = xn + dn;
        X[i] = xf;
        bad |= !isfinite(xf);
      } else {
        X[i] = xn;
        S.R[i] = r;
        S.D[i] = dn;
      }
    });
  }
}

template <int K>
__global__ void __launch_bounds__(CV_NT, 1) coarse_vcycle_kernel(const __grid_constant__ SpkCoarseArgs a) {
  constexpr int W = 2 * K + 1, NC = K + 2;
  __shared__ double bm[NC * W], bk[NC * W];
  extern __shared__ double sm[];
  const int blk = blockIdx.x;
  const int lc = a.lc;
  // shared memory: the operator's four sweep buffers at the top level's size and every vector of the
  // levels below lc; level lc's x and b are the caller's arrays and r, d, w (all levels) live in a
  // per-block global scratch -- L2-resident, so the top level may be larger than the smem budget
  // would allow for all nine of its vectors
  CVShared S;
  S.dim = a.dim;
  const int nmax = CVLevel<K>(lc, a.dim).n;
  double* p = sm;
  S.T0 = p; p += nmax;
  S.T1 = p; p += nmax;
  S.T2 = p; p += nmax;
  S.T3 = p; p += nmax;
  for (int l = 0; l < lc; ++l) {
    const CVLevel<K> L(l, a.dim);
    S.X[l] = p; p += L.n;
    S.B[l] = p; p += L.n;
  }
  for (int l = 1; l <= lc; ++l) {
    S.DI[l] = p;
    p += CVLevel<K>(l, a.dim).n;
  }
  {
    int* ip = reinterpret_cast<int*>(p);
    for (int l = 0; l <= lc; ++l) {
      const CVLevel<K> L(l, a.dim);
      for (int i = threadIdx.x; i < L.n; i += CV_NT) {
        const int z = i % L.m, t = i / L.m, y = t % L.m, x = t / L.m;
        ip[i] = x | (y << 10) | (z << 20);
      }
      S.CO[l] = ip;
      ip += L.n;
    }
  }
  // the top level's x, b, r, d, w: in shared memory when they fit (every access of the cycle's many
  // short phases then avoids an L2 round trip; measured: the 2D C1 cycle), else in global memory
  double* xg = a.x + (long long)blk * a.sx;
  const double* bg = a.b + (long long)blk * a.sb;
  const bool top_smem = a.top_in_smem != 0;
  {
    int* ip = reinterpret_cast<int*>(p);
    int ints = 0;
    for (int l = 0; l <= lc; ++l) ints += CVLevel<K>(l, a.dim).n;
    p = reinterpret_cast<double*>(ip) + (ints + 1) / 2;  // past the coordinate tables
  }
  if (top_smem) {
    S.X[lc] = p; p += nmax;
    S.B[lc] = p; p += nmax;
    S.R = p; p += nmax;
    S.D = p; p += nmax;
    S.W = p; p += nmax;
  } else {
    S.X[lc] = xg;
    S.B[lc] = const_cast<double*>(bg);
    double* scr = a.scratch + (long long)blk * 3 * nmax;
    S.R = scr;
    S.D = scr + nmax;
    S.W = scr + 2 * nmax;
  }
  S.bm = bm;
  S.bk = bk;
  Band<K>::build(bm, bk);
  spk_pdl_wait();
  if (top_smem)
    for (int i = threadIdx.x; i < nmax; i += CV_NT) S.B[lc][i] = bg[i];
  __syncthreads();
  const double lam = a.lam[blk];
  for (int l = 1; l <= lc; ++l) {
    const CVLevel<K> L(l, a.dim);
    const double lamp = lam * a.hd[l], taup = a.tau * a.hk[l];
    for (int i = threadIdx.x; i < L.n; i += CV_NT) {
      const int z = i % L.m, t = i / L.m, y = t % L.m, x = t / L.m;
      S.DI[l][i] = cv_dinv<K>(x, y, z, L.m, L.mx, lamp, taup);
    }
  }
  __syncthreads();
  bool bad[SPK_CV_LMAX + 1];
#pragma unroll
  for (int l = 0; l <= SPK_CV_LMAX; ++l) bad[l] = false;
  // down: pre-smoothing from zero, residual, restriction
  for (int l = lc; l >= 1; --l) {
    const double lamp = lam * a.hd[l], taup = a.tau * a.hk[l];
    cv_smooth<K>(S, a, l, blk, true, lamp, taup, bad[l]);
    const double* Bl = S.B[l];
    cv_apply<K>(S, l, S.X[l], lamp, taup, [&](int i, double w) { S.R[i] = Bl[i] - w; });
    cv_restrict<K>(S, a.P, l);
  }
  // coarse: x_0 = Cinv b_0 (dense inverse of the assembled constrained operator)
  {
    const int n0 = CVLevel<K>(0, a.dim).n;
    const double* C = a.cinv + (long long)blk * n0 * n0;
    for (int i = threadIdx.x; i < n0; i += CV_NT) {
      double acc = 0.0;
      for (int j = 0; j < n0; ++j) acc = fma(C[(long long)i * n0 + j], S.B[0][j], acc);
      S.X[0][i] = acc;
    }
    __syncthreads();
  }
  // up: prolongation (accumulate), post-smoothing from the current iterate
  for (int l = 1; l <= lc; ++l) {
    const double lamp = lam * a.hd[l], taup = a.tau * a.hk[l];
    cv_prolong<K>(S, a.P, l);
    cv_smooth<K>(S, a, l, blk, false, lamp, taup, bad[l]);
  }
  if (top_smem) {
    for (int i = threadIdx.x; i < nmax; i += CV_NT) xg[i] = S.X[lc][i];
  }
  spk_pdl_trigger();  // at the end: dependents parked early would share this CTA's SM for its whole run
  if (a.flags) {
    for (int l = 1; l <= lc; ++l)
      if (bad[l]) atomicOr(a.flags + l, 1);
  }
}

}  // namespace

long long spk_coarse_vcycle_top_bytes(int K, int lc, int dim) {
  const long long m = ((long long)K << lc) + 1;
  return 5 * (dim == 3 ? m * m * m : m * m) * (long long)sizeof(double);
}

long long spk_coarse_vcycle_smem(int K, int lc, int dim) {
  auto nodes = [&](int l) {
    const long long m = ((long long)K << l) + 1;
    return dim == 3 ? m * m * m : m * m;
  };
  long long tot = 0;
  for (int l = 0; l < lc; ++l) tot += 2 * nodes(l);
  for (int l = 1; l <= lc; ++l) tot += nodes(l);  // Jacobi tables
  long long ints = 0;
  for (int l = 0; l <= lc; ++l) ints += nodes(l);  // coordinate tables
  tot += (ints + 1) / 2;
  return (tot + 4 * nodes(lc)) * (long long)sizeof(double);
}

cudaError_t spk_launch_coarse_vcycle(int K, const SpkCoarseArgs& a, cudaStream_t s) {
  const long long bytes = spk_coarse_vcycle_smem(K, a.lc, a.dim) +
                          (a.top_in_smem ? spk_coarse_vcycle_top_bytes(K, a.lc, a.dim) : 0);
  if (a.lc < 1 || a.lc > SPK_CV_LMAX || bytes > SPK_CV_SMEM_MAX) return cudaErrorInvalidValue;
  switch (K) {
#define SPK_CV(KK)                                                                                   \
  case KK: {                                                                                         \
    static bool cfg = false;                                                                         \
    if (!cfg) {                                                                                      \
      cudaError_t e = cudaFuncSetAttribute(coarse_vcycle_kernel<KK>,                                 \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, SPK_CV_SMEM_MAX); \
      if (e != cudaSuccess) return e;                                                                \
      cfg = true;                                                                                    \
    }                                                                                                \
    return spk_launch(coarse_vcycle_kernel<KK>, dim3(a.nblk), dim3(CV_NT), (size_t)bytes, s, a);     \
  }
    SPK_CV(1) SPK_CV(2) SPK_CV(3) SPK_CV(4)
#undef SPK_CV
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
