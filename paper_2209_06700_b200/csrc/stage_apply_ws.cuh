// K1w: warp-specialised form of K1 (stage_apply.cuh) for 3D levels, sm_100a, fp64.
//
// Same operator, same (y, z) tile x x-chunk decomposition and the same fused epilogues as K1
// (reference fem.py:120-170 through the Kronecker form, see stage_apply.cuh), but the three sweeps of
// a plane are owned by different warps that run as a producer / consumer chain over shared-memory
// rings guarded by mbarriers -- there is no CTA-wide barrier in the plane loop:
//
//   producer (1 warp)  TMA: one 2D box per (stage, row parity) of plane t -> U ring   (UTMALDG)
//   Z warps            a = Mz u, b = Kz u          U ring  -> (A, B) ring
//   Y warps            ma = My a, c = Ky a + My b  (A, B)  -> (MA, C) ring
//   X warps            stage mix + element-push accumulation in registers, fused epilogue
//
// Why: K1's per-thread Z -> Y -> X sequence puts every warp of the CTA in the same phase at the same
// time (a shared-memory burst, then a DFMA burst), so the two pipes alternate instead of overlapping:
// measured shared-memory time + FP64 time ~ elapsed time (profiles/r02_stage_apply_ncu_summary.txt).
// With one role per warp the SM always holds warps in different phases, the Z / Y items are half
// rows / half columns (13 loads per 8 outputs instead of 9 per 4), and the plane loads leave the
// instruction stream (6 TMA boxes per plane instead of ~1300 8-byte cp.async).
//
// TMA and the reference layout: a level's row stride is n_ax * 8 bytes with n_ax = k 2^l + 1 odd, not
// a legal tensor-map stride (16-byte multiples). Two rows are: the maps describe the vector as
//   dim0 = flat element index (stage, plane, row parity and z offset folded into the coordinate)
//   dim1 = row PAIR index inside the plane, stride 2 * nz * 8 bytes, exact size (y bounds -> zero fill)
// so a plane's rows arrive as an even-row box and an odd-row box. Odd rows are fetched one element
// early; that one-double skew makes 16 consecutive rows of the (even-pitch) boxes hit 16 distinct
// shared-memory banks in the Z sweep. Boxes of tiles at the high z edge start at nz - W so that no
// box crosses the end of the array.
#pragma once
#include <cuda.h>

#ifndef SPK_WS_SETREG
#define SPK_WS_SETREG 1
#endif
#ifndef SPK_WS_REG_ZY
#define SPK_WS_REG_ZY 56
#endif
#ifndef SPK_WS_NXW
#define SPK_WS_NXW 4
#endif
#ifndef SPK_ROLE
#define SPK_ROLE(r) true
#endif
namespace {

template <int K, int Q> struct WGeo {
  using G = Geo<K, Q>;
  static constexpr int TYE = G::TYE, TZE = G::TZE, TY = G::TY, TZ = G::TZ;
  static_assert(TY * TZ <= 256, "one X thread per tile node");
  static constexpr int NYin = TY + K + 1, NZin = TZ + K + 1;
  static constexpr int TZp = TZ | 1;
#ifdef SPK_WS_NZW
  static constexpr int NZW = SPK_WS_NZW, NYW = SPK_WS_NYW;
#else
  static constexpr int NZW = 4, NYW = 3;
#endif
  static constexpr int NXW = SPK_WS_NXW;  // X warps: 256 / (32 NXW) tile nodes per thread
  static constexpr int NT = 32 * (NZW + NYW + 1 + NXW);
  static constexpr int YW0 = NZW, PW = NZW + NYW, XW0 = NZW + NYW + 1;
  static constexpr int W = G::W, BOXR = G::BOXR, REG = G::REG;  // TMA boxes: see Geo
  static constexpr int U_SLOT = Q * 2 * REG;             // doubles
  static constexpr int AB_SLOT = 2 * Q * NYin * TZp;
  static constexpr int MC_SLOT = 2 * Q * TY * TZp;
  static constexpr int DT_SZ = G::DT_SZ;
  static constexpr int bytes(int nu, int nab, int nmc) {
    return 8 * (nu * U_SLOT + nab * AB_SLOT + nmc * MC_SLOT + DT_SZ) + 256;
  }
  static constexpr int LIM2 = 113 * 1024;  // two CTAs per SM
  static constexpr int NU = bytes(3, 2, 3) <= LIM2 ? 3 : 2;
  static constexpr int NAB = 2;
  static constexpr int NMC = bytes(NU, 2, 3) <= LIM2 ? 3 : 2;
  static constexpr int SMEM_BYTES = bytes(NU, NAB, NMC);
#ifdef SPK_WS_MINB
  static constexpr int MINB = SPK_WS_MINB;
#else
  static constexpr int MINB = SMEM_BYTES <= LIM2 ? 2 : 1;
#endif
  // Z items: (stage, row, half row); Y items: (stage, z, half column)
  static constexpr int ZS = (TZE + 1) / 2, ZSEG = (TZE + ZS - 1) / ZS;
  static constexpr int YS = (TYE + 1) / 2, YSEG = (TYE + YS - 1) / YS;
  static constexpr int ZITEMS = Q * ZSEG * NYin, NZT = 32 * NZW, ZIT = (ZITEMS + NZT - 1) / NZT;
  static constexpr int YITEMS = Q * YSEG * TZ, NYT = 32 * NYW, YIT = (YITEMS + NYT - 1) / NYT;
  // setmaxnreg works on warpgroups: warps 0-3 (Z), 4-7 (Y + producer), 8-15 (X)
  // (launch bound 384 threads x 2 CTAs -> 80 registers per thread = 240 per lane of the three
  // warpgroups; Z and Y + producer keep REG_ZY each, X takes the rest)
  static constexpr bool SETREG = SPK_WS_SETREG && (NZW == 4 && NYW == 3 && NXW == 4 && MINB == 2);
  static constexpr int REG_ZY = SPK_WS_REG_ZY, REG_X = 240 - 2 * REG_ZY;
  static constexpr unsigned TX_BYTES = 2u * Q * BOXR * W * 8u;
};

// named barriers (producer / consumer between roles: the waiting warps block in hardware instead of
// polling an mbarrier; ids 1..15, count = arriving + waiting threads)
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
// (the documented PTX producer pattern: st.shared ; bar.arrive  /  bar.sync ; ld.shared -- the
// barrier orders the participating threads' prior shared-memory accesses)
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <int K, int Q, bool BLOCK, int EPI, bool FULL>
__device__ __forceinline__ void stage_apply_ws_body(const SpkApplyArgs& a, const SpkWsMaps& maps, double* smem) {
  using G = WGeo<K, Q>;
  using H = Hat<K>;
  constexpr int TYE = G::TYE, TZE = G::TZE, TY = G::TY, TZ = G::TZ;
  constexpr int NYin = G::NYin, TZp = G::TZp, W = G::W, REG = G::REG;
  constexpr int NU = G::NU, NAB = G::NAB, NMC = G::NMC;

  double* Us = smem;                          // [NU][Q][2][REG]
  double* ABs = Us + NU * G::U_SLOT;          // [NAB][Q][NYin][TZp] of (A, B)
  double* MCs = ABs + NAB * G::AB_SLOT;       // [NMC][Q][TY][TZp] of (MA, C)
  double* dtab = MCs + NMC * G::MC_SLOT;      // Jacobi table
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(dtab + G::DT_SZ);
  unsigned long long* u_full = bars;            // [NU]   producer -> Z
  unsigned long long* u_empty = u_full + NU;    // [NU]   Z -> producer
  // named barriers: (A, B) ring Z <-> Y, (MA, C) ring Y <-> X
  constexpr int B_AB_FULL = 1, B_AB_EMPTY = B_AB_FULL + NAB, B_MC_FULL = B_AB_EMPTY + NAB, B_MC_EMPTY = B_MC_FULL + NMC;
  static_assert(B_MC_EMPTY + NMC <= 16, "16 named barriers per CTA");
  constexpr int N_ZY = 32 * (G::NZW + G::NYW), N_YX = 32 * (G::NYW + G::NXW);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const SpkDims g = a.g;
  const int ez0 = blockIdx.x * TZE, ey0 = blockIdx.y * TYE;
  const int chunk = blockIdx.z % a.nchunks;
  const int b0 = BLOCK ? (a.blk_base + (int)(blockIdx.z / a.nchunks) * Q) : 0;
  const int z_lo = K * ez0, z_hi = min(K * (ez0 + TZE), g.nz);
  const int y_lo = K * ey0, y_hi = min(K * (ey0 + TYE), g.ny);
  const int nzo = FULL ? TZ : z_hi - z_lo, nyo = FULL ? TY : y_hi - y_lo;
  const int nez = FULL ? TZE : min(TZE, g.Ez + 1 - ez0);
  const int ney = FULL ? TYE : min(TYE, g.Ey + 1 - ey0);

  double lamq[Q], ith[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    lamq[q] = BLOCK ? (a.lam_uniform ? a.lam[0] : a.lam[b0 - a.blk_base + q]) : 0.0;
    ith[q] = 1.0 / a.c2[BLOCK ? b0 - a.blk_base + q : 0];
  }
  if constexpr (EPI != EPI_STORE) {
    constexpr int K1 = K + 1;
    for (int idx = tid; idx < K1 * K1 * K1; idx += G::NT) {
      const int cx = idx / (K1 * K1), cy = (idx / K1) % K1, cz = idx % K1;
      double mx, kx, my, ky, mz, kz;
      class_diag1<K>(cx, g.Ex, mx, kx);
      class_diag1<K>(cy, g.Ey, my, ky);
      class_diag1<K>(cz, g.Ez, mz, kz);
      const double dm = (mx * my) * mz;
      const double dk = ((kx * my) * mz + (mx * ky) * mz) + (mx * my) * kz;
      double* e = dtab + idx * Geo<K, Q>::DT_STRIDE;
      if constexpr (BLOCK) {
#pragma unroll
        for (int q = 0; q < Q; ++q) e[q] = 1.0 / (lamq[q] * dm + a.tau * dk);
      } else {
        const double da = a.jre * dm + a.tau * dk, db = a.jim * dm;
        const double det = da * da + db * db;
        e[0] = da / det;
        e[1] = db / det;
      }
    }
  }

  // x-chunk (elements [ex0, ex1)); planes K*ecur .. K*ex1 (as K1)
  const int ex0 = a.ex_begin + chunk * a.xe_chunk;
  const int ex1 = min(a.ex_end, ex0 + a.xe_chunk);
  const int efirst = g.x0 < 0 ? -g.x0 / K : 0;
  int ecur = (ex0 > efirst) ? ex0 - 1 : ex0;
  const int xs = K * ecur;
  const int nplanes = K * ex1 - xs + 1;
  const long long plane_stride = (long long)g.ny * g.nz;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      mbar_init(&u_full[i], 1);
      mbar_init(&u_empty[i], G::NZW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  spk_pdl_wait();  // everything above reads parameters / constants only

  // Box start along z. TMA needs a 16-byte aligned start address, i.e. an even flat element index
  // from the (16-byte aligned) map base: the start is the flat index of the tile's first loaded node
  // rounded down to even, so a row's values sit at offset 0 or 1 of its box row (`par`). Rows are an
  // odd number of doubles apart, so the even- and the odd-row box get opposite offsets: 16
  // consecutive rows of the (even-pitch) boxes hit 16 distinct banks in the Z sweep. A box that would
  // cross the row end starts at nz - W instead, rounded UP to even (`clamped`: it may then read the
  // one double that shares the last row's final 16-byte chunk; the Z sweep never uses it).
  const bool clamped = z_lo - K + W > g.nz;
  const int zoff = clamped ? g.nz - W : z_lo - K;
  const int dlc = clamped ? (z_lo - K) - (g.nz - W) : 0;
  const long long base0 = (BLOCK ? (long long)b0 * a.su : 0) + maps.bias;
  const int ye = y_lo - K;  // first loaded global row

  // Register budget per role (setmaxnreg works on warpgroups, and the allocator honours it only inside
  // the branch it dominates): the launch bound gives 80 registers per thread; the Z and the Y +
  // producer warpgroups shrink to REG_ZY and the X warpgroup, which holds the x accumulators of two
  // nodes per thread, grows to REG_X.
  if (warp >= G::YW0 && warp < G::XW0) {
    if constexpr (G::SETREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(G::REG_ZY));
  if (SPK_ROLE(0) && warp == G::PW) {
    // ---------------- producer: TMA boxes of plane t into U slot t % NU ----------------
    if (lane == 0) {
      // loaded row yy is global row ye + yy and lives in box (yy & 1); the even map holds the even
      // global rows (pair index gy / 2), the odd map the odd ones (pair index (gy - 1) / 2, + nz)
      const int r0e = (ye & 1) ? ye + 1 : ye, r0o = (ye & 1) ? ye : ye + 1;
      const int c1e = r0e >> 1, c1o = (r0o - 1) >> 1;  // arithmetic shifts: floor
      const int be = (r0e - ye) & 1, bo = (r0o - ye) & 1;
      for (int t = 0; t < nplanes; ++t) {
        const int s = t % NU;
        mbar_wait(&u_empty[s], ((t / NU) & 1) ^ 1);
        mbar_arrive_expect_tx(&u_full[s], G::TX_BYTES);
        double* Ub = Us + s * G::U_SLOT;
        const long long pb = base0 + (long long)(xs + t) * plane_stride + zoff;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const long long fe = pb + (long long)q * a.su, fo = fe + g.nz;
          const long long ce = clamped ? (fe + 1) & ~1LL : fe & ~1LL, co = clamped ? (fo + 1) & ~1LL : fo & ~1LL;
          tma_box_2d(Ub + (q * 2 + be) * REG, &maps.even, (int)ce, c1e, &u_full[s]);
          tma_box_2d(Ub + (q * 2 + bo) * REG, &maps.odd, (int)co, c1o, &u_full[s]);
        }
      }
    }
  } else if (SPK_ROLE(2)) {
    // ---------------- Y warps: (MA, C) = (My A, Ky A + My B) ----------------
    const int ytid = tid - 32 * G::YW0;
    int yab[G::YIT], ymc[G::YIT], yeb[G::YIT];
#pragma unroll
    for (int i = 0; i < G::YIT; ++i) {
      const int it = ytid + i * G::NYT;
      yeb[i] = TYE;
      yab[i] = 0;
      ymc[i] = 0;
      if (it < G::YITEMS) {
        const int zl = it % TZ, rest = it / TZ;
        const int seg = rest % G::YSEG, q = rest / G::YSEG;
        if (zl < nzo) {
          yeb[i] = seg * G::YS;
          yab[i] = (q * NYin) * TZp + zl;
          ymc[i] = (q * TY) * TZp + zl;
        }
      }
    }
    for (int t = 0; t < nplanes; ++t) {
      const int ab = t % NAB, mc = t % NMC;
      nbar_sync(B_AB_FULL + ab, N_ZY);
      if (t >= NMC) nbar_sync(B_MC_EMPTY + mc, N_YX);
      const double2* AB = reinterpret_cast<const double2*>(ABs + ab * G::AB_SLOT);
      double2* MC = reinterpret_cast<double2*>(MCs + mc * G::MC_SLOT);
#pragma unroll
      for (int i = 0; i < G::YIT; ++i) {
        const int e_beg = yeb[i];
        if (e_beg >= ney) continue;
        const double2* col = AB + yab[i] + (K * e_beg) * TZp;
        double2* out = MC + ymc[i] + (K * e_beg) * TZp;
        double2 R[K + 1];
#pragma unroll
        for (int s2 = 0; s2 <= K; ++s2) R[s2] = col[s2 * TZp];
        double cm = 0.0, cc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 <= K; ++s2) {
          cm = fma(H::M(K, s2), R[s2].x, cm);
          cc = fma(H::S(K, s2), R[s2].x, cc);
          cc = fma(H::M(K, s2), R[s2].y, cc);
        }
#pragma unroll
        for (int el = 0; el < G::YS; ++el) {
          const int e = e_beg + el;
          if (e < ney) {
            R[0] = R[K];
#pragma unroll
            for (int s2 = 1; s2 <= K; ++s2) R[s2] = col[(K * el + K + s2) * TZp];
            const int ey = ey0 + e;
            const double wl = (FULL || ey > 0) ? 1.0 : 0.0, wr = (FULL || ey < g.Ey) ? 1.0 : 0.0;
            double rm = 0.0, rc = 0.0;
#pragma unroll
            for (int s2 = 0; s2 <= K; ++s2) {
              rm = fma(H::M(0, s2), R[s2].x, rm);
              rc = fma(H::S(0, s2), R[s2].x, rc);
              rc = fma(H::M(0, s2), R[s2].y, rc);
            }
            out[(K * el) * TZp] = make_double2(fma(wl, cm, wr * rm), fma(wl, cc, wr * rc));
#pragma unroll
            for (int r = 1; r < K; ++r) {
              double am = 0.0, ac = 0.0;
#pragma unroll
              for (int s2 = 0; s2 <= K; ++s2) {
                am = fma(H::M(r, s2), R[s2].x, am);
                ac = fma(H::S(r, s2), R[s2].x, ac);
                ac = fma(H::M(r, s2), R[s2].y, ac);
              }
              out[(K * el + r) * TZp] = make_double2(am, ac);
            }
            if (el + 1 < G::YS) {
              cm = 0.0;
              cc = 0.0;
#pragma unroll
              for (int s2 = 0; s2 <= K; ++s2) {
                cm = fma(H::M(K, s2), R[s2].x, cm);
                cc = fma(H::S(K, s2), R[s2].x, cc);
                cc = fma(H::M(K, s2), R[s2].y, cc);
              }
            }
          }
        }
      }
      nbar_arrive(B_MC_FULL + mc, N_YX);
      nbar_arrive(B_AB_EMPTY + ab, N_ZY);
    }
  }
  } else if (SPK_ROLE(1) && warp < G::NZW) {
    if constexpr (G::SETREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(G::REG_ZY));
    // ---------------- Z warps: (A, B) = (Mz u, Kz u) ----------------
    int zrow[G::ZIT], zab[G::ZIT], zeb[G::ZIT];
    unsigned zpar = 0u;  // bit i: parity of item i's box start index at plane 0
    const unsigned podd = static_cast<unsigned>(plane_stride & 1);
#pragma unroll
    for (int i = 0; i < G::ZIT; ++i) {
      const int it = tid + i * G::NZT;
      zeb[i] = TZE;
      zrow[i] = 0;
      zab[i] = 0;
      if (it < G::ZITEMS) {
        // rows 0..15 of every (stage, segment) first (half-warps on 16 consecutive rows: distinct
        // banks for the loads and the 16-byte stores), then the remaining rows
        constexpr int R = NYin < 16 ? NYin : 16, QS = Q * G::ZSEG, T = NYin - R;
        int yy, qs;
        if (it < QS * R) {
          qs = it / R;
          yy = it - qs * R;
        } else {
          const int idx = it - QS * R;
          qs = idx / (T > 0 ? T : 1);
          yy = R + idx - qs * T;
        }
        const int q = qs / G::ZSEG, seg = qs - q * G::ZSEG;
        const int gy = ye + yy;
        zeb[i] = seg * G::ZS;
        zrow[i] = (q * 2 + (yy & 1)) * REG + (yy >> 1) * W + dlc;
        const long long f0 = base0 + (long long)q * a.su + (long long)xs * plane_stride + ((gy & 1) ? g.nz : 0) + zoff;
        zpar |= static_cast<unsigned>(f0 & 1) << i;
        zab[i] = (q * NYin + yy) * TZp;
        // constrained: y-boundary rows are zero rows (the boxes hold the raw values)
        if (!FULL && a.constrained && (gy == 0 || gy == g.ny - 1)) zeb[i] = -1 - zeb[i];
      }
    }
    for (int t = 0; t < nplanes; ++t) {
      const int s = t % NU, ab = t % NAB;
      mbar_wait(&u_full[s], (t / NU) & 1);
      if (t >= NAB) nbar_sync(B_AB_EMPTY + ab, N_ZY);
      const double* Ub = Us + s * G::U_SLOT;
      double2* AB = reinterpret_cast<double2*>(ABs + ab * G::AB_SLOT);
      const int xg = xs + t + g.x0;
      const bool xzero = a.constrained && (xg == 0 || xg == g.nxg - 1);
#pragma unroll
      for (int i = 0; i < G::ZIT; ++i) {
        const bool rowzero = !FULL && zeb[i] < 0;
        const int e_beg = rowzero ? -1 - zeb[i] : zeb[i];
        if (e_beg >= nez) continue;
        double2* abrow = AB + zab[i] + K * e_beg;
        if (xzero || rowzero) {
#pragma unroll
          for (int el = 0; el < G::ZS; ++el)
            if (e_beg + el < nez) {
#pragma unroll
              for (int r = 0; r < K; ++r) abrow[K * el + r] = make_double2(0.0, 0.0);
            }
          continue;
        }
        const int par = static_cast<int>(((zpar >> i) ^ (static_cast<unsigned>(t) & podd)) & 1u);
        const double* row = Ub + zrow[i] + K * e_beg + (clamped ? -par : par);
        // node index of row[0] along z (FULL: unused)
        const int zb = z_lo - K + K * e_beg;
        const int zmin = a.constrained ? 1 : 0, zmax = g.nz - 1 - zmin;  // valid (non-zero) input nodes
        auto ld = [&](int j) -> double {
          if constexpr (FULL) return row[j];
          const int zi = zb + j;
          return (zi >= zmin && zi <= zmax) ? row[j] : 0.0;
        };
        double R[K + 1];
#pragma unroll
        for (int s2 = 0; s2 <= K; ++s2) R[s2] = ld(s2);
        double ca = 0.0, cb = 0.0;  // row K of the element left of the segment (shared vertex)
#pragma unroll
        for (int s2 = 0; s2 <= K; ++s2) {
          ca = fma(H::M(K, s2), R[s2], ca);
          cb = fma(H::S(K, s2), R[s2], cb);
        }
#pragma unroll
        for (int el = 0; el < G::ZS; ++el) {
          const int e = e_beg + el;
          if (e < nez) {
            R[0] = R[K];
#pragma unroll
            for (int s2 = 1; s2 <= K; ++s2) R[s2] = ld(K * el + K + s2);
            const int ez = ez0 + e;
            const double wl = (FULL || ez > 0) ? 1.0 : 0.0, wr = (FULL || ez < g.Ez) ? 1.0 : 0.0;
            double r1 = 0.0, r2 = 0.0;
#pragma unroll
            for (int s2 = 0; s2 <= K; ++s2) {
              r1 = fma(H::M(0, s2), R[s2], r1);
              r2 = fma(H::S(0, s2), R[s2], r2);
            }
            abrow[K * el] = make_double2(fma(wl, ca, wr * r1), fma(wl, cb, wr * r2));
#pragma unroll
            for (int r = 1; r < K; ++r) {
              double a1 = 0.0, a2 = 0.0;
#pragma unroll
              for (int s2 = 0; s2 <= K; ++s2) {
                a1 = fma(H::M(r, s2), R[s2], a1);
                a2 = fma(H::S(r, s2), R[s2], a2);
              }
              abrow[K * el + r] = make_double2(a1, a2);
            }
            if (el + 1 < G::ZS) {
              ca = 0.0;
              cb = 0.0;
#pragma unroll
              for (int s2 = 0; s2 <= K; ++s2) {
                ca = fma(H::M(K, s2), R[s2], ca);
                cb = fma(H::S(K, s2), R[s2], cb);
              }
            }
          }
        }
      }
      nbar_arrive(B_AB_FULL + ab, N_ZY);
      __syncwarp();
      if (lane == 0) mbar_arrive(&u_empty[s]);
    }
  } else if (SPK_ROLE(3) && warp >= G::XW0) {
    if constexpr (G::SETREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(G::REG_X));
    // ---------------- X warps: stage mix + element push + fused epilogue ----------------
    constexpr int NXT = 32 * G::NXW, PPT = (TY * TZ + NXT - 1) / NXT;
    const int xt = tid - 32 * G::XW0;
    int yy[PPT], zz[PPT], mcoff[PPT];
    long long pyz[PPT];
    bool pv[PPT];
    double acc[PPT][Q][K + 1];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int p = xt + j * NXT;
      const int yl = p / TZ, zl = p - yl * TZ;
      pv[j] = (p < TY * TZ) && (FULL || (yl < nyo && zl < nzo));
      yy[j] = y_lo + yl;
      zz[j] = z_lo + zl;
      pyz[j] = (long long)yy[j] * g.nz + zz[j];
      mcoff[j] = pv[j] ? yl * TZp + zl : 0;
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int s2 = 0; s2 <= K; ++s2) acc[j][q][s2] = 0.0;
    }
    double sumsq = 0.0;
    const bool dm_ident = a.dm_identity != 0;

    // One copy of the plane step for every local plane index r_loc (uniform): the x-table column is
    // read from the constant bank at run time. (Five compile-time copies -- times two nodes, times
    // the inlined epilogue -- overflow the instruction cache once the roles run different code:
    // measured no_instruction stall 3.3 warps per issue.)
    auto xstep = [&](auto JC, int r_loc, const double (&cm)[K + 1], const double (&ck)[K + 1],
                     const double (&ma)[Q], const double (&cc)[Q]) {
      constexpr int j = decltype(JC)::value;
      double pq[Q], qq[Q];
      if constexpr (BLOCK) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          pq[q] = fma(lamq[q], ma[q], a.tau * cc[q]);
          qq[q] = a.tau * ma[q];
        }
      } else {
        if (dm_ident) {
#pragma unroll
          for (int i = 0; i < Q; ++i) {
            double pp = a.DM[i][i] * ma[i], s3 = 0.0;
#pragma unroll
            for (int jj = 0; jj < Q; ++jj) {
              pp = fma(a.DK[i][jj], cc[jj], pp);
              s3 = fma(a.DK[i][jj], ma[jj], s3);
            }
            pq[i] = pp;
            qq[i] = s3;
          }
        } else {
#pragma unroll
          for (int i = 0; i < Q; ++i) {
            double pp = 0.0, s3 = 0.0;
#pragma unroll
            for (int jj = 0; jj < Q; ++jj) {
              pp = fma(a.DM[i][jj], ma[jj], pp);
              pp = fma(a.DK[i][jj], cc[jj], pp);
              s3 = fma(a.DK[i][jj], ma[jj], s3);
            }
            pq[i] = pp;
            qq[i] = s3;
          }
        }
      }
#pragma unroll
      for (int s2 = 0; s2 <= K; ++s2)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[j][q][s2] = fma(cm[s2], pq[q], fma(ck[s2], qq[q], acc[j][q][s2]));
      if (r_loc == K) {
        if (ecur >= ex0) {
#pragma unroll
          for (int s2 = 0; s2 < K; ++s2) {
            double val[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) val[q] = acc[j][q][s2];
            const int xx = K * ecur + s2;
            epilogue<K, Q, BLOCK, EPI, FULL>(a, b0, lamq, dtab, ith, xx, yy[j], zz[j],
                                             (long long)xx * plane_stride + pyz[j], val, sumsq);
          }
        }
        if (ecur + 1 == g.Ex && a.store_last) {
          double val[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) val[q] = acc[j][q][K];
          epilogue<K, Q, BLOCK, EPI, FULL>(a, b0, lamq, dtab, ith, K * g.Ex, yy[j], zz[j],
                                           (long long)(K * g.Ex) * plane_stride + pyz[j], val, sumsq);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double carry = acc[j][q][K];
#pragma unroll
          for (int s2 = 0; s2 <= K; ++s2) acc[j][q][s2] = fma(H::M(s2, 0), pq[q], H::S(s2, 0) * qq[q]);
          acc[j][q][0] += carry;
        }
      }
    };

    for (int t = 0; t < nplanes; ++t) {
      const int mc = t % NMC;
      nbar_sync(B_MC_FULL + mc, N_YX);
      const double2* MC = reinterpret_cast<const double2*>(MCs + mc * G::MC_SLOT);
      double ma[PPT][Q], cc[PPT][Q];
#pragma unroll
      for (int j = 0; j < PPT; ++j)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const double2 v2 = MC[mcoff[j] + (q * TY) * TZp];  // (lanes without a node read slot 0)
          ma[j][q] = v2.x;
          cc[j][q] = v2.y;
        }
      nbar_arrive(B_MC_EMPTY + mc, N_YX);
      const int r_loc = xs + t - K * ecur;  // 0..K, uniform
      double cm[K + 1], ck[K + 1];  // symmetric tables: row r_loc = column r_loc
#pragma unroll
      for (int s2 = 0; s2 <= K; ++s2) {
        cm[s2] = c_hat[K - 1][0][r_loc][s2];
        ck[s2] = c_hat[K - 1][1][r_loc][s2];
      }
      if (pv[0]) xstep(IC<0>{}, r_loc, cm, ck, ma[0], cc[0]);
      if constexpr (PPT > 1)
        if (pv[1]) xstep(IC<1>{}, r_loc, cm, ck, ma[PPT > 1 ? 1 : 0], cc[PPT > 1 ? 1 : 0]);
      static_assert(PPT <= 2, "X nodes per thread");
      if (r_loc == K) ++ecur;
    }
  }
  spk_pdl_trigger();
}

template <int K, int Q, bool BLOCK, int EPI>
__global__ void __launch_bounds__(WGeo<K, Q>::NT, WGeo<K, Q>::MINB)
    stage_apply_ws_kernel(const __grid_constant__ SpkApplyArgs a, const __grid_constant__ SpkWsMaps maps) {
  extern __shared__ __align__(128) double smem_ws[];
  using G = WGeo<K, Q>;
  const SpkDims& g = a.g;
  const int ez0 = blockIdx.x * G::TZE, ey0 = blockIdx.y * G::TYE;
  const int lo = a.constrained ? 2 : 1, hi = a.constrained ? 1 : 0;
  const bool full = ey0 >= lo && ez0 >= lo && ey0 + G::TYE + hi <= g.Ey && ez0 + G::TZE + hi <= g.Ez;
  if (full) stage_apply_ws_body<K, Q, BLOCK, EPI, true>(a, maps, smem_ws);
  else stage_apply_ws_body<K, Q, BLOCK, EPI, false>(a, maps, smem_ws);
}

// ---- host: tensor maps ----
typedef CUresult (*SpkEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline SpkEncodeTiled spk_encode_tiled() {
  static SpkEncodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<SpkEncodeTiled>(p);
  }
  return fn;
}

// whether K1w can take this launch, and its tensor maps
template <int K, int Q>
bool ws_maps(const SpkApplyArgs& a, bool block, SpkWsMaps* m) {
  using G = Geo<K, Q>;
  const SpkDims& g = a.g;
  m->bias = -1;
  if (g.Ex <= 0 || g.Ey <= 0 || g.Ez <= 0) return false;
  SpkEncodeTiled enc = spk_encode_tiled();
  if (!enc) return false;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(a.u);
  if (addr & 7) return false;
  const uintptr_t base = addr & ~uintptr_t(15);
  m->bias = (int)((addr - base) >> 3);
  const long long stages = block ? (long long)a.blk_base + a.nblk : Q;
  const long long total = m->bias + (stages - 1) * a.su + g.n;
  if (total >= (1LL << 31) - 4096 || a.su < 0) return false;
  const cuuint64_t stride[1] = {(cuuint64_t)g.nz * 16};
  const cuuint32_t box[2] = {(cuuint32_t)G::W, (cuuint32_t)G::BOXR};
  const cuuint32_t estr[2] = {1, 1};
  for (int par = 0; par < 2; ++par) {
    const cuuint64_t dims[2] = {(cuuint64_t)total, (cuuint64_t)((g.ny + 1 - par) / 2)};
    if (dims[1] == 0) return false;
    CUresult r = enc(par ? &m->odd : &m->even, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, reinterpret_cast<void*>(base),
                     dims, stride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

template <int K, int Q, bool BLOCK, int EPI>
cudaError_t launch_ws(const SpkApplyArgs& a, const SpkWsMaps& maps, cudaStream_t s, int* nctas_out) {
  using G = WGeo<K, Q>;
  static bool configured = false;
  auto kern = stage_apply_ws_kernel<K, Q, BLOCK, EPI>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int gz = (a.g.Ez + 1 + G::TZE - 1) / G::TZE;
  const int gy = (a.g.Ey + 1 + G::TYE - 1) / G::TYE;
  const int nb = BLOCK ? a.nblk / Q : 1;
  dim3 grid(gz, gy, a.nchunks * nb);
  if (nctas_out) *nctas_out = gz * gy * a.nchunks * nb;
  return spk_launch(kern, grid, dim3(G::NT), (size_t)G::SMEM_BYTES, s, a, maps);
}

}  // namespace
