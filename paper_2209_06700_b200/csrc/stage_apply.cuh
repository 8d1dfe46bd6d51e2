// K1: batched / stage-coupled matrix-free Q_k operator on the uniform grid, sm_100a, fp64.
//
//   coupled mode : v_i = sum_j ( DM_ij M + DK_ij K ) u_j        i,j < Q      (I(x)M + tau A(x)K, ...)
//   block mode   : v_b = lam_b M u_b + tau K u_b                 b < nblk     (lam M + tau K per block)
//
// M = Mx(x)My(x)Mz and K = Kx My Mz + Mx Ky Mz + Mx My Kz are the Kronecker forms the reference
// applies with dense 1D contractions (fem.py:120-151, _contract fem.py:37-41). Here the assembled
// 1D matrices are never formed: each axis is applied element-by-element from the (k+1)x(k+1)
// reference-element tables (compile-time constants, spk_tables.cuh), which is the flop-minimal
// banded form (SURVEY.md §7 hard part 1). The mesh size is folded into the stage mix:
// M = h^d M_hat, K = h^(d-2) K_hat, so the host passes DM' = h^d DM and DK' = h^(d-2) DK.
//
// Schedule ("2.5D sliding window", one CTA = one (y,z) tile x one x-chunk, all Q stages):
//   per x-plane:  plane x+1 into the other smem buffer (double buffering): TMA boxes completing on an
//                 mbarrier for interior tiles (load_plane_tma), per-node cp.async with zero-fill for
//                 the ragged tiles on the high side
//                 Z-phase   a = Mz u, b = Kz u                 (smem -> smem, 2 elements / item)
//                 Y-phase   ma = My a, c = Ky a + My b          (smem -> smem, 2 elements / item)
//                 X-phase   stage mix p_i = sum_j DM_ij ma_j + DK_ij c_j, q_i = sum_j DK_ij ma_j
//                           and element-push accumulation v += Mx[.,r] p + Kx[.,r] q in registers
//   an element's K output planes are finished when its last plane arrives -> fused epilogue.
// Every thread's work items are fixed for the whole kernel (no per-plane index arithmetic).
// HBM traffic per apply: read u once (+ L2-resident halo), write v once = 16 B per stage-DoF.
#pragma once
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <type_traits>
#include "spk_internal.cuh"
#include "spk_tables.cuh"
#include <cuda.h>

#ifndef SPK_MINB_ALL
#define SPK_MINB_ALL 1
#endif
// Split plane barrier: each thread arrives on an mbarrier once its Z(t) / Y(t-1) results (and its
// cp.async of plane t+1) are in shared memory, THEN runs X(t-2), and waits for the others' arrivals
// only at the start of the next interval, so the X-phase of the warps with the most Z/Y work overlaps
// the next interval of the others (MA/C triple-buffered for it).
#ifndef SPK_SPLIT_BAR
#define SPK_SPLIT_BAR 1
#endif
// TMA plane loads for interior tiles (two 2D boxes per stage and plane, see load_plane_tma)
#ifndef SPK_WARP_ARRIVE
#define SPK_WARP_ARRIVE 0   // measured: no gain (C2 388.3 vs 387.8 us)
#endif
#ifndef SPK_TMA_LOAD
#define SPK_TMA_LOAD 1
#endif
// Balanced Z map (k = 4, Q = 3, 256 threads): the 192 Y items occupy six of the eight warps, so with
// one Z item per thread the two Y-less warps idle for ~40 % of every plane interval. Here the Y-less
// warps take two whole Z items each and the other Z items are split into half-element items (output
// rows {0, 1} / {2, 3}) spread over the six Y warps: per-warp DFMA work per interval 159 / 164 / 170
// instead of 105 / 184.
// MEASURED AND REJECTED (off): bitwise identical results, barrier waits down (long-scoreboard stall
// 1.06 -> 0.84 per issue), but C2 went 365 -> 466 us: warps of one scheduler now run different Z code
// and miss in the instruction cache (no_instruction stall 0.36 -> 1.37 per issue), even with the
// smaller runtime-index X-phase (424 us). profiles/r02_k1_ab.txt
#ifndef SPK_ZBAL
#define SPK_ZBAL 0
#endif
// K1's hot loop is large enough to miss in the instruction cache (ncu: no_instruction stalls); knobs
// that trade compile-time constants for footprint
#ifndef SPK_SPLIT_UNROLL2
#define SPK_SPLIT_UNROLL2 1
#endif
// (measured: one interval copy with runtime buffer parity loses, C2 369 -> 387 us; one X-phase copy
// with the x-table column read from constant memory by the plane index wins, C2 369 -> 364 us,
// constrained 415 -> 404 us)
#ifndef SPK_XR_RUNTIME
#define SPK_XR_RUNTIME 1
#endif
// EPI_STORE elements without identity rows are written with plain streaming stores (no per-node tests)
#ifndef SPK_FAST_STORE
#define SPK_FAST_STORE 1
#endif

namespace {

template <int K> struct Tile;
// (y, z) tiles of ~256 output nodes: one 256-thread CTA owns one node per thread in the X-phase and
// two CTAs fit on an SM (registers and shared memory), so one CTA's barrier waits overlap the
// other's work (measured on B200: 16x16 tiles, 2 CTAs/SM beat 16x32 tiles, 1 CTA/SM by ~8 %)
template <> struct Tile<1> { static constexpr int TYE = 16, TZE = 16; };
template <> struct Tile<2> { static constexpr int TYE = 8, TZE = 8; };
template <> struct Tile<3> { static constexpr int TYE = 5, TZE = 5; };
#ifndef SPK_K4_TZE
#define SPK_K4_TZE 4
#endif
template <> struct Tile<4> { static constexpr int TYE = 4, TZE = SPK_K4_TZE; };

#ifndef SPK_Q1_TILE
#define SPK_Q1_TILE 1
#endif
template <int K, int Q> struct Geo {
  // one stage / block per CTA leaves most threads idle in the Z / Y phases of a ~256-node tile:
  // Q = 1 sweeps a SPK_Q1_TILE^2 larger tile (several X points per thread)
  static constexpr int TSC = (Q == 1) ? SPK_Q1_TILE : 1;
  static constexpr int TYE = Tile<K>::TYE * TSC, TZE = Tile<K>::TZE * TSC;
  static constexpr int TY = K * TYE, TZ = K * TZE;
  // 1 barrier per plane: Z, Y, X run on three plane buffers (see the pipeline below)
  static constexpr bool PIPE3 = true;
  static constexpr int NT = (Q >= 2 && TY * TZ > 256) ? 512 : (TY * TZ < 256 && TY * TZ > 128 ? (TY * TZ + 31) / 32 * 32 : 256);
  static constexpr int NBUF = PIPE3 ? 2 : 1;
  static constexpr int NYin = TY + K + 1, NZin = TZ + K + 1;
  static constexpr int NZp = NZin | 1;   // odd pitch: lanes walking rows hit distinct banks
  static constexpr int TZp = TZ | 1;
  // TMA layout of a plane buffer (interior tiles): per stage an even-row and an odd-row box of BOXR
  // rows x W doubles (see load_plane_tma). W: even (16-byte multiple), >= NZin + 1 (a row's values sit
  // at offset 0 or 1 of its box row), W / 2 odd (16 consecutive rows hit 16 distinct banks)
  static constexpr int wpitch() {
    int w = (NZin + 2) & ~1;
    while ((w / 2) % 2 == 0) w += 2;
    return w;
  }
  static constexpr int W = wpitch();
  static constexpr int BOXR = (NYin + 1) / 2;
  static constexpr int REG = (BOXR * W + 15) / 16 * 16;  // one box, 128-byte multiple
  static constexpr int U_SZT = Q * 2 * REG;
  static constexpr unsigned TX_BYTES = 2u * Q * BOXR * W * 8u;
  static constexpr int U_SZ = (SPK_TMA_LOAD && U_SZT > Q * NYin * NZp) ? U_SZT : Q * NYin * NZp;  // one plane buffer
  static constexpr int AB_SZ = Q * NYin * TZp;         // one of A / B
  static constexpr int MC_SZ = Q * TY * TZp;           // one of MA / C
  // Jacobi table: one entry per (x,y,z) node class ((K+1)^3) and block (block mode) / (A, B) (pair)
  static constexpr int DT_STRIDE = (Q > 2 ? Q : 2);
  static constexpr int DT_SZ = (K + 1) * (K + 1) * (K + 1) * DT_STRIDE;
  // split barrier (SPK_SPLIT_BAR) where it was measured to pay (profiles/r02_k1_ab.txt): k = 4
  // (C2 426 -> 408 us); at k = 2 / 3 it lost 2-32 % (at k = 2, Q = 4 the third (MA, C) buffer also
  // pushes the CTA past two per SM)
  static constexpr int SMEM_SPLIT = 2 * U_SZ + 2 * NBUF * AB_SZ + 2 * 3 * MC_SZ + DT_SZ + 4;
  static constexpr bool SPLIT = SPK_SPLIT_BAR && K == 4 && NT <= 256 &&
                                (NT == 256 ? SMEM_SPLIT * 8 <= 112 * 1024 : SMEM_SPLIT * 8 <= 74 * 1024);
  static constexpr int MCBUF = SPLIT ? 3 : NBUF;  // (MA, C) plane buffers
  static constexpr int SMEM_DOUBLES = 2 * U_SZ + 2 * NBUF * AB_SZ + 2 * MCBUF * MC_SZ + DT_SZ + 4;  // + mbarriers
  static constexpr int PPT = (TY * TZ + NT - 1) / NT;
  // Z items: (q, yy, element segment), ZS elements per segment
#ifdef SPK_ZS
  static constexpr int ZS = (Q >= 2) ? SPK_ZS : 1;
#else
  static constexpr int ZS = 1;
#endif
  static constexpr int ZSEG = (TZE + ZS - 1) / ZS;
  static constexpr int ZITEMS = Q * NYin * ZSEG;
  static constexpr int ZIT = (ZITEMS + NT - 1) / NT;
  // balanced Z map (SPK_ZBAL): two item slots per thread, each a whole item or a half item
  static constexpr bool ZBAL = SPK_ZBAL && K == 4 && Q == 3 && NT == 256 && ZS == 1 && TYE == 4 && TZE == 4;
  static constexpr int ZSLOTS = ZBAL ? 2 : ZIT;
  // Y items: (q, z, element segment)
#ifdef SPK_YS
  static constexpr int YS = (Q >= 2) ? SPK_YS : 1;
#else
  static constexpr int YS = 1;
#endif
  static constexpr int YSEG = (TYE + YS - 1) / YS;
  static constexpr int YITEMS = Q * TZ * YSEG;
  static constexpr int YIT = (YITEMS + NT - 1) / NT;
  // U load items
  static constexpr int LITEMS = Q * NYin * NZin;
  static constexpr int LIT = (LITEMS + NT - 1) / NT;
  static_assert(LIT <= 32, "load items are flagged in one 32-bit mask");
// Low degrees sweeping one or two blocks per CTA fit four CTAs per SM (64 registers, <= 55 KB): twice
// the warps to hide the plane pipeline's latency (measured: C4 block STORE 531 -> 484 us with two
// blocks per CTA). SPK_MINB4 = highest degree that gets the 4-CTA launch bound.
#ifndef SPK_MINB4
#define SPK_MINB4 3
#endif
  static constexpr bool MINB4_OK = SPK_MINB4 && K <= SPK_MINB4 && NT <= 256 && SMEM_DOUBLES * 8 <= 55 * 1024;
  static constexpr int MINB = (NT <= 192 && SMEM_DOUBLES * 8 <= 74 * 1024)   ? 3
                              : (NT <= 256 && SMEM_DOUBLES * 8 <= 112 * 1024) ? 2
                                                                              : 1;
};

// Distinct entries of a symmetric, centro-symmetric (K+1)x(K+1) element table:
// (r,s) ~ (s,r) ~ (K-r,K-s) ~ (K-s,K-r). cls() maps an entry to its class, NC classes in total.
template <int K> struct Sym {
  __host__ __device__ static constexpr int canon(int r, int s) {
    int best = r * 16 + s;
    const int c2 = s * 16 + r, c3 = (K - r) * 16 + (K - s), c4 = (K - s) * 16 + (K - r);
    if (c2 < best) best = c2;
    if (c3 < best) best = c3;
    if (c4 < best) best = c4;
    return best;
  }
  __host__ __device__ static constexpr int cls(int r, int s) {
    const int me = canon(r, s);
    int n = 0;
    for (int a = 0; a <= K; ++a)
      for (int b = 0; b <= K; ++b)
        if (canon(a, b) == a * 16 + b && a * 16 + b < me) ++n;
    return n;
  }
  __host__ __device__ static constexpr int count() {
    int n = 0;
    for (int a = 0; a <= K; ++a)
      for (int b = 0; b <= K; ++b)
        if (canon(a, b) == a * 16 + b) ++n;
    return n;
  }
};

// reference-element mass (M) and stiffness (S) tables held in registers
template <int K> struct Coef {
  static constexpr int NC = Sym<K>::count();
  double mv[NC], sv[NC];
  __device__ __forceinline__ void load() {
#pragma unroll
    for (int r = 0; r <= K; ++r)
#pragma unroll
      for (int s = 0; s <= K; ++s) {
        mv[Sym<K>::cls(r, s)] = c_hat[K - 1][0][r][s];
        sv[Sym<K>::cls(r, s)] = c_hat[K - 1][1][r][s];
      }
  }
  __device__ __forceinline__ double m(int r, int s) const { return mv[Sym<K>::cls(r, s)]; }
  __device__ __forceinline__ double s(int r, int s2) const { return sv[Sym<K>::cls(r, s2)]; }
};

template <int V> struct IC { static constexpr int value = V; };
// plane-buffer parity: a compile-time IC<p> (unrolled pipeline) or a runtime int
template <int V> __device__ __forceinline__ constexpr int parity_of(IC<V>) { return V; }
__device__ __forceinline__ int parity_of(int v) { return v; }
template <int V> __device__ __forceinline__ constexpr IC<1 - V> other_parity(IC<V>) { return {}; }
__device__ __forceinline__ int other_parity(int v) { return 1 - v; }

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// ---- Blackwell bulk-async copies (the TMA engine's non-tensor path: UBLKCP) completing on an
//      mbarrier transaction count (SYNCS) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Waiting on an mbarrier costs issue slots: K1 is bound by its non-DFMA instructions (the FP64 pipe
// takes a DFMA every other cycle per scheduler and ~1 other instruction per DFMA is free, tools/
// ubench/fp64_mix.cu), and try_wait with a suspend-time hint still woke the waiting warps ~15 times
// per wait (17 % of K1's issued instructions were its polling loop: profiles/r02_k1_final_ncu.txt).
// SPK_WAIT_NS > 0: test once, then sleep SPK_WAIT_NS between tests.
#ifndef SPK_WAIT_NS
#define SPK_WAIT_NS 0
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
#if SPK_WAIT_NS > 0
  asm volatile(
      "{\n .reg .pred p;\n"
      "SPK_MBAR_WAIT_%=:\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @p bra SPK_MBAR_DONE_%=;\n"
      " nanosleep.u32 %2;\n"
      " bra SPK_MBAR_WAIT_%=;\n"
      "SPK_MBAR_DONE_%=:\n}\n" ::"r"(smem_u32(bar)), "r"(phase), "r"((unsigned)SPK_WAIT_NS)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n"
      "SPK_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra SPK_MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase), "r"(0x989680u)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// TMA plane loads and the reference layout. A level's row stride is n_ax * 8 bytes with n_ax = k 2^l + 1
// odd -- not a legal tensor-map stride (16-byte multiples) -- but TWO rows are. The maps describe the
// vector as  dim0 = flat element index from the 16-byte aligned base (stage, plane, row parity and z
// offset go into the coordinate),  dim1 = row PAIR index inside a plane (stride 2 nz 8 bytes, exact
// size: rows outside the plane are zero-filled), so a plane of a stage arrives as an even-row box
// and an odd-row box of BOXR x W doubles. The box start must be 16-byte aligned (an odd start
// coordinate traps: tools/ubench/tma_probe.cu), so it is the flat index of the tile's first loaded
// node rounded down to even and a row's values sit at offset 0 or 1 of its box row; rows are an odd
// number of doubles apart, so the two boxes get opposite offsets and 16 consecutive rows of the
// (even-pitch) boxes hit 16 distinct banks in the Z sweep. One thread issues the 2 Q boxes of a
// plane (SASS: UTMALDG.2D); they complete on the plane buffer's mbarrier.
// (Round-2 history: one 176-byte cp.async.bulk per ROW, 63 per plane, ran C2 at 711 us and was
// rejected: profiles/r02_k1_ab.txt.)
struct SpkWsMaps {
  CUtensorMap even, odd;
  int bias;  // elements between the 16-byte aligned map base and args.u (0 or 1); < 0: no maps
};

__device__ __forceinline__ void tma_box_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// assembled 1D reference diagonal at node i of an axis with E elements (E == 0: degenerate axis)
template <int K>
__device__ __forceinline__ void diag1(int i, int E, double& dm, double& dk) {
  using H = Hat<K>;
  if (E == 0) { dm = 1.0; dk = 0.0; return; }
  const int e = i / K, r = i - e * K;
  if (r != 0) {
    double m = 0.0, s = 0.0;
#pragma unroll
    for (int rr = 1; rr < K; ++rr)
      if (rr == r) { m = H::M(rr, rr); s = H::S(rr, rr); }
    dm = m; dk = s;
    return;
  }
  dm = 0.0; dk = 0.0;
  if (e > 0) { dm += H::M(K, K); dk += H::S(K, K); }
  if (e < E) { dm += H::M(0, 0); dk += H::S(0, 0); }
}

// reference-element diagonal pieces at a node (association order of np.multiply.outer chains,
// reference fem.py:172-187); the caller scales by DM' / DK'
template <int K>
__device__ __forceinline__ void node_diag(const SpkDims& g, int x, int y, int z, double& dm, double& dk) {
  double mx, kx, my, ky, mz, kz;
  diag1<K>(x, g.Ex, mx, kx);
  diag1<K>(y, g.Ey, my, ky);
  diag1<K>(z, g.Ez, mz, kz);
  dm = (mx * my) * mz;
  dk = ((kx * my) * mz + (mx * ky) * mz) + (mx * my) * kz;
}

// Node class along one axis for the Jacobi table: 0 interior vertex, 1..K-1 element-interior node,
// K boundary vertex (the assembled 1D diagonal takes K+1 distinct values). Degenerate axis: 0.
template <int K>
__device__ __forceinline__ int axis_class(int i, int n, int E) {
  if (E == 0) return 0;
  const int r = i % K;
  if (r != 0) return r;
  return (i == 0 || i == n - 1) ? K : 0;
}

template <int K>
__device__ __forceinline__ void class_diag1(int c, int E, double& dm, double& dk) {
  using H = Hat<K>;
  if (E == 0) { dm = 1.0; dk = 0.0; return; }
  if (c == 0) { dm = H::M(K, K) + H::M(0, 0); dk = H::S(K, K) + H::S(0, 0); return; }
  if (c == K) { dm = H::M(0, 0); dk = H::S(0, 0); return; }
  double m = 0.0, s2 = 0.0;
#pragma unroll
  for (int rr = 1; rr < K; ++rr)
    if (rr == c) { m = H::M(rr, rr); s2 = H::S(rr, rr); }
  dm = m;
  dk = s2;
}

__device__ __forceinline__ bool on_boundary(const SpkDims& g, int x, int y, int z) {
  return (g.Ex > 0 && (x + g.x0 == 0 || x + g.x0 == g.nxg - 1)) || (g.Ey > 0 && (y == 0 || y == g.ny - 1)) ||
         (g.Ez > 0 && (z == 0 || z == g.nz - 1));
}

// z-sweep of one element: vertex r=0 gathers the left element (row K) and the right element
// (row 0); interior r>=1 use the right element only. Outputs a = M_hat u, b = K_hat u.
template <int K>
__device__ __forceinline__ void elem2(const Coef<K>& cf, const double (&L)[K + 1], const double (&R)[K + 1],
                                      double wl, double wr, double (&o1)[K], double (&o2)[K]) {
  double l1 = 0.0, l2 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
  for (int s = 0; s <= K; ++s) {
    l1 = fma(cf.m(K, s), L[s], l1);
    l2 = fma(cf.s(K, s), L[s], l2);
    r1 = fma(cf.m(0, s), R[s], r1);
    r2 = fma(cf.s(0, s), R[s], r2);
  }
  o1[0] = fma(wl, l1, wr * r1);
  o2[0] = fma(wl, l2, wr * r2);
#pragma unroll
  for (int r = 1; r < K; ++r) {
    double a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int s = 0; s <= K; ++s) {
      a1 = fma(cf.m(r, s), R[s], a1);
      a2 = fma(cf.s(r, s), R[s], a2);
    }
    o1[r] = a1;
    o2[r] = a2;
  }
}

// half-element forms of elem2 (balanced Z map): FIRST = output rows [0, K/2) (the vertex row needs the
// left element), !FIRST = rows [K/2, K) (right element only); outputs land in o1 / o2 [0, K/2)
template <int K, bool FIRST>
__device__ __forceinline__ void elem2_half(const Coef<K>& cf, const double (&L)[K + 1], const double (&R)[K + 1],
                                           double wl, double wr, double (&o1)[K / 2], double (&o2)[K / 2]) {
  constexpr int H = K / 2;
  if constexpr (FIRST) {
    double l1 = 0.0, l2 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
    for (int s = 0; s <= K; ++s) {
      l1 = fma(cf.m(K, s), L[s], l1);
      l2 = fma(cf.s(K, s), L[s], l2);
      r1 = fma(cf.m(0, s), R[s], r1);
      r2 = fma(cf.s(0, s), R[s], r2);
    }
    o1[0] = fma(wl, l1, wr * r1);
    o2[0] = fma(wl, l2, wr * r2);
  }
#pragma unroll
  for (int r = FIRST ? 1 : H; r < (FIRST ? H : K); ++r) {
    double a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int s = 0; s <= K; ++s) {
      a1 = fma(cf.m(r, s), R[s], a1);
      a2 = fma(cf.s(r, s), R[s], a2);
    }
    o1[FIRST ? r : r - H] = a1;
    o2[FIRST ? r : r - H] = a2;
  }
}

// y-sweep of one element on two inputs: ma = M_hat a ; c = K_hat a + M_hat b
template <int K>
__device__ __forceinline__ void elem3(const Coef<K>& cf, const double (&La)[K + 1],
                                      const double (&Ra)[K + 1], const double (&Lb)[K + 1],
                                      const double (&Rb)[K + 1], double wl, double wr, double (&ma)[K],
                                      double (&c)[K]) {
  double lm = 0.0, lc = 0.0, rm = 0.0, rc = 0.0;
#pragma unroll
  for (int s = 0; s <= K; ++s) {
    lm = fma(cf.m(K, s), La[s], lm);
    lc = fma(cf.s(K, s), La[s], lc);
    lc = fma(cf.m(K, s), Lb[s], lc);
    rm = fma(cf.m(0, s), Ra[s], rm);
    rc = fma(cf.s(0, s), Ra[s], rc);
    rc = fma(cf.m(0, s), Rb[s], rc);
  }
  ma[0] = fma(wl, lm, wr * rm);
  c[0] = fma(wl, lc, wr * rc);
#pragma unroll
  for (int r = 1; r < K; ++r) {
    double am = 0.0, ac = 0.0;
#pragma unroll
    for (int s = 0; s <= K; ++s) {
      am = fma(cf.m(r, s), Ra[s], am);
      ac = fma(cf.s(r, s), Ra[s], ac);
      ac = fma(cf.m(r, s), Rb[s], ac);
    }
    ma[r] = am;
    c[r] = ac;
  }
}

// Fused epilogue at one node for all Q stages / blocks of the CTA. Block mode: stage q of the CTA is
// block b0 + q with its own shift lam[q] (and Chebyshev coefficients in its parameter slot).
template <int K, int Q, bool BLOCK, int EPI, bool FULL = false>
__device__ __forceinline__ void epilogue(const SpkApplyArgs& a, int b0, const double (&lamq)[Q],
                                         const double* dtab, const double (&ith)[Q], int x, int y, int z,
                                         long long gi, const double (&val)[Q], double& sumsq,
                                         int qfirst = 0) {
  // gi: node index of (x, y, z) in the level (x * ny*nz + y * nz + z), precomputed by the caller.
  // Virtual x-split: stage q of the CTA sits q*vplanes planes further along x (its global x differs).
  // Stages q < qfirst are skipped (the last vertex plane of a virtual range belongs to the next).
  const SpkDims& g = a.g;
  const long long ubase = (BLOCK ? (long long)b0 * a.su : 0) + gi;
  const long long ebase = (BLOCK ? (long long)b0 * a.se : 0) + gi;
  const long long vbase = (BLOCK ? (long long)b0 * a.sv : 0) + gi;
  const int slot0 = BLOCK ? b0 - a.blk_base : 0;
  const bool vsplit = BLOCK && a.vplanes != 0;
  const bool bnd_yz = !FULL && a.constrained && ((g.Ey > 0 && (y == 0 || y == g.ny - 1)) ||
                                                 (g.Ez > 0 && (z == 0 || z == g.nz - 1)));
  bool bndq[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int xg = x + g.x0 + (vsplit ? q * a.vplanes : 0);
    bndq[q] = bnd_yz || (a.constrained && g.Ex > 0 && (xg == 0 || xg == g.nxg - 1));
  }
  bool bnd = false;
#pragma unroll
  for (int q = 0; q < Q; ++q) bnd |= bndq[q];
  double Av[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) Av[q] = val[q];
  if (bnd) {  // constrained boundary rows are the identity (rare: a real branch, not a select)
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (bndq[q]) Av[q] = __ldg(a.u + ubase + q * a.su);
  }

  if constexpr (EPI == EPI_STORE) {
    double* vp = a.v + vbase;
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (q >= qfirst) __stcs(vp + q * a.sv, Av[q]);
  } else {
    // Jacobi diagonal (reference operator_diagonal fem.py:172-187, 1.0 on boundary): looked up in
    // the per-CTA table of node classes (no per-node division)
    constexpr int K1 = K + 1;
    const int cyz = axis_class<K>(y, g.ny, g.Ey) * K1 + axis_class<K>(z, g.nz, g.Ez);
    const int cls = axis_class<K>(x + g.x0, g.nxg, g.Ex) * K1 * K1 + cyz;
    const double* dt = dtab + cls * Geo<K, Q>::DT_STRIDE;
    double z0[Q];  // Dinv applied to the quantity of the epilogue
    auto jacobi = [&](const double (&rr)[Q]) {
      if constexpr (BLOCK) {
        if (vsplit) {  // per-stage x class (one block: table column 0)
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int cq = axis_class<K>(x + g.x0 + q * a.vplanes, g.nxg, g.Ex) * K1 * K1 + cyz;
            z0[q] = (bndq[q] ? 1.0 : dtab[cq * Geo<K, Q>::DT_STRIDE]) * rr[q];
          }
        } else {
#pragma unroll
          for (int q = 0; q < Q; ++q) z0[q] = (bndq[q] ? 1.0 : dt[q]) * rr[q];
        }
      } else {  // pair 2x2 block Jacobi (multigrid.py:268-276, 306-313)
        const double A_ = bnd ? 1.0 : dt[0], B_ = bnd ? 0.0 : dt[1];
        z0[0] = A_ * rr[0] + B_ * rr[1];
        if constexpr (Q > 1) z0[1] = -B_ * rr[0] + A_ * rr[1];
      }
    };
    double* rp = a.r + ebase;
    double* xp = a.x + ebase;
    if constexpr (EPI == EPI_DINV) {
      jacobi(Av);
      double* vp = a.v + vbase;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (q < qfirst) continue;
        vp[q * a.sv] = z0[q];
        sumsq = fma(z0[q], z0[q], sumsq);
      }
    } else {
      double rn[Q], xfin[Q], dq[Q];
      if constexpr (EPI == EPI_RESID) {
        const double* bp = a.b + ebase;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          rn[q] = __ldg(bp + q * a.se) - Av[q];
          if (q >= qfirst) rp[q * a.se] = rn[q];
        }
      } else {  // EPI_CHEB:  x += d ; r -= A d ; d = c1 d + c2 Dinv r   (multigrid.py:82-87)
        const double* up = a.u + ubase;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          dq[q] = __ldg(up + q * a.su);
          rn[q] = rp[q * a.se] - Av[q];
          const double xq = xp[q * a.se] + dq[q];
          if (!a.final_step) {
            if (q >= qfirst) {
              rp[q * a.se] = rn[q];
              xp[q * a.se] = xq;
            }
          } else {
            xfin[q] = xq;
          }
        }
      }
      if (a.d_out != nullptr) {
        jacobi(rn);
        bool bad = false;
        double* dp = a.d_out + ebase;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int slot = BLOCK ? slot0 + q : 0;
          double dn;
          if constexpr (EPI == EPI_CHEB) {
            dn = a.c1[slot] * dq[q] + a.c2[slot] * z0[q];
            if (a.final_step) {  // last step fused with "return x + d" (multigrid.py:88) + NaN check
              const double xn = xfin[q] + dn;
              if (q >= qfirst) {
                xp[q * a.se] = xn;
                bad |= !isfinite(xn);
              }
              continue;
            }
          } else {
            dn = z0[q] * ith[q];  // post-smoothing start: d = (Dinv r) / theta  (multigrid.py:77)
          }
          if (q >= qfirst) dp[q * a.se] = dn;
        }
        if (bad && a.nan_flag) atomicOr(a.nan_flag, 1);
      }
    }
  }
}

// FULL: the CTA's (y, z) tile and its loaded halo lie strictly inside the domain (no zero-filled
// slots, no missing neighbour elements, no constrained y/z boundary rows): every per-item bound
// check and boundary weight is compile-time (measured: the predicate / select overhead of the
// generic body is a visible share of K1's issue slots).
// FULLV: 0 generic tile; 1 interior tile; 2 interior tile on the low y / z boundary (the missing
// element gets weight 0 in the Z / Y sweeps, boundary rows are identity rows in the epilogue)
template <int K, int Q, bool BLOCK, int EPI, int FULLV>
__device__ __forceinline__ void stage_apply_body(const SpkApplyArgs& a, const SpkWsMaps& maps, double* smem) {
  constexpr bool FULL = FULLV != 0, LOW = FULLV == 2;
  using G = Geo<K, Q>;
  constexpr int TYE = G::TYE, TZE = G::TZE, TY = G::TY, TZ = G::TZ, NT = G::NT;
  constexpr int NYin = G::NYin, NZin = G::NZin, NZp = G::NZp, TZp = G::TZp;
  constexpr int PPT = G::PPT;

  double* Us = smem;                    // [2][Q][NYin][NZp]
  double* ABs = Us + 2 * G::U_SZ;       // [2][Q][NYin][TZp] of (A, B) pairs (16-byte accesses)
  double* MCs = ABs + 2 * G::NBUF * G::AB_SZ;  // [NBUF][Q][TY][TZp] of (MA, C) pairs
  double* dtab = MCs + 2 * G::MCBUF * G::MC_SZ;  // [(K+1)^3][DT_STRIDE] Jacobi table
  unsigned long long* ubar = reinterpret_cast<unsigned long long*>(dtab + G::DT_SZ);  // plane-buffer mbarriers
  unsigned long long* ibar = ubar + 2;  // split plane barrier (SPK_SPLIT_BAR)
  // interior tiles load their planes with TMA boxes (issued by thread 0) that complete on
  // ubar[slot]; every other tile keeps the per-node cp.async path with zero-fill
  constexpr bool BULK = FULL && SPK_TMA_LOAD;

  const int tid = threadIdx.x;
  const SpkDims g = a.g;
  const bool ydeg = !FULL && (g.Ey == 0), xdeg = !FULL && (g.Ex == 0);
  const int ez0 = blockIdx.x * TZE, ey0 = blockIdx.y * TYE;
  const int chunk = blockIdx.z % a.nchunks;
  const int b0 = BLOCK ? (a.blk_base + (int)(blockIdx.z / a.nchunks) * Q) : 0;  // first block of CTA

  const int z_lo = K * ez0, z_hi = min(K * (ez0 + TZE), g.nz);
  const int y_lo = ydeg ? 0 : K * ey0, y_hi = ydeg ? 1 : min(K * (ey0 + TYE), g.ny);
  const int nzo = FULL ? TZ : z_hi - z_lo, nyo = FULL ? TY : y_hi - y_lo;
  const int nez = FULL ? TZE : min(TZE, g.Ez + 1 - ez0);  // includes the virtual last-vertex element
  const int ney = FULL ? TYE : (ydeg ? 1 : min(TYE, g.Ey + 1 - ey0));
  const double* __restrict__ u = a.u + (BLOCK ? (long long)b0 * a.su : 0);

  double lamq[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) lamq[q] = BLOCK ? (a.lam_uniform ? a.lam[0] : a.lam[b0 - a.blk_base + q]) : 0.0;
  double ith[Q];  // 1 / theta per block (post-smoothing start)
#pragma unroll
  for (int q = 0; q < Q; ++q) ith[q] = 1.0 / a.c2[BLOCK ? b0 - a.blk_base + q : 0];
  if constexpr (EPI != EPI_STORE) {
    constexpr int K1 = K + 1;
    for (int idx = tid; idx < K1 * K1 * K1; idx += NT) {
      const int cx = idx / (K1 * K1), cy = (idx / K1) % K1, cz = idx % K1;
      double mx, kx, my, ky, mz, kz;
      class_diag1<K>(cx, g.Ex, mx, kx);
      class_diag1<K>(cy, g.Ey, my, ky);
      class_diag1<K>(cz, g.Ez, mz, kz);
      const double dm = (mx * my) * mz;
      const double dk = ((kx * my) * mz + (mx * ky) * mz) + (mx * my) * kz;
      double* e = dtab + idx * G::DT_STRIDE;
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

  // reference-element tables in registers (distinct entries only)
  Coef<K> cf;
  cf.load();

  // x-chunk (elements [ex0, ex1)); planes K*(ex0-1) .. K*ex1
  int ex0 = 0, ex1 = 0, xs = 0, nplanes = 1, ecur = 0;
  if (!xdeg) {
    ex0 = a.ex_begin + chunk * a.xe_chunk;
    ex1 = min(a.ex_end, ex0 + a.xe_chunk);
    // first real element of the window (a first slab has padding planes x0 < 0 in front); with a
    // virtual x-split every range starts one element early (the left neighbour range's last
    // element, zero-filled for the first range)
    const int efirst = g.x0 < 0 ? -g.x0 / K : 0;
    ecur = (ex0 > efirst || (BLOCK && a.vplanes)) ? ex0 - 1 : ex0;
    xs = K * ecur;
    nplanes = K * ex1 - xs + 1;
  }

  // ---- fixed per-thread work descriptors ----
  const long long plane_stride = (long long)g.ny * g.nz;
  // U-plane load items, fixed for the kernel: a 32-bit source byte offset (from u), the shared
  // address, and one bit of `lzero` per item = zero-fill (slots outside the domain and, constrained,
  // y/z-boundary nodes). One 8-byte cp.async per item and plane whose ignore-src predicate writes
  // the zeros; no branches, no per-plane index math beyond one 64-bit add.
  unsigned loff[BULK ? 1 : G::LIT], ldst[BULK ? 1 : G::LIT];
  unsigned lzero = 0u;
  unsigned lq[Q];  // virtual x-split: items of stage q (their global x is q*vplanes further)
#pragma unroll
  for (int q = 0; q < Q; ++q) lq[q] = 0u;
  constexpr bool LTAIL = (G::LITEMS % NT) != 0;  // only the last item can be past the end
  if constexpr (!BULK) {
#pragma unroll
    for (int i = 0; i < G::LIT; ++i) {
      const int idx = min(tid + i * NT, G::LITEMS - 1);
      const int q = idx / (NYin * NZin);
      const int rem = idx - q * (NYin * NZin);
      const int yy = rem / NZin, zz = rem - yy * NZin;
      const int gy = y_lo - K + yy, gz = z_lo - K + zz;
      const int slot = (q * NYin + yy) * NZp + zz;
      ldst[i] = static_cast<unsigned>(__cvta_generic_to_shared(Us + slot));
      const bool in = gy >= 0 && gy < g.ny && gz >= 0 && gz < g.nz;
      const bool bnd = (!ydeg && (gy == 0 || gy == g.ny - 1)) || gz == 0 || gz == g.nz - 1;
      loff[i] = (FULL || in) ? static_cast<unsigned>((q * a.su + (long long)gy * g.nz + gz) * 8) : 0u;
      if (!FULL && (!in || (a.constrained && bnd))) lzero |= 1u << i;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq)
        if (q == qq) lq[qq] |= 1u << i;
    }
  }
  constexpr unsigned UBUF = G::U_SZ * sizeof(double);

  unsigned bpar0 = 0u;  // bit i: parity of Z item i's box start index at plane 0
  const unsigned podd = static_cast<unsigned>(plane_stride & 1);
  auto load_plane_tma = [&](int x, auto BUF) {
    const unsigned buf = parity_of(BUF);
    if (tid != 0) return;
    double* Ub = Us + buf * G::U_SZ;
    mbar_arrive_expect_tx(&ubar[buf], G::TX_BYTES);
    // loaded row yy is global row ye + yy and lives in box (yy & 1); the even map holds the even
    // global rows (pair index gy / 2), the odd map the odd ones (pair index (gy - 1) / 2, + nz)
    const int ye = y_lo - K;
    const int r0e = (ye & 1) ? ye + 1 : ye, r0o = (ye & 1) ? ye : ye + 1;
    const int c1e = r0e >> 1, c1o = (r0o - 1) >> 1;
    const int be = (r0e - ye) & 1, bo = (r0o - ye) & 1;
    const long long pb = (BLOCK ? (long long)b0 * a.su : 0) + maps.bias + (long long)x * plane_stride + (z_lo - K);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const long long fe = pb + (long long)q * a.su, fo = fe + g.nz;
      tma_box_2d(Ub + (q * 2 + be) * G::REG, &maps.even, (int)(fe & ~1LL), c1e, &ubar[buf]);
      tma_box_2d(Ub + (q * 2 + bo) * G::REG, &maps.odd, (int)(fo & ~1LL), c1o, &ubar[buf]);
    }
  };

  auto load_plane = [&](int x, auto BUF) {
    if constexpr (BULK) {
      load_plane_tma(x, BUF);
      return;
    }
    const unsigned buf = parity_of(BUF);
    const unsigned long long base =
        reinterpret_cast<unsigned long long>(u) + (unsigned long long)x * (unsigned long long)plane_stride * 8ull;
    // constrained: the x-boundary planes are zero (uniform per plane); virtual x-split: per stage,
    // and planes left of the domain (first range's halo element) are zero too
    unsigned zmask = lzero;
    if (BLOCK && a.vplanes) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int xg = x + g.x0 + q * a.vplanes;
        if (xg < 0 || (a.constrained && (xg == 0 || xg == g.nxg - 1))) zmask |= lq[q];
      }
    } else {
      const bool xb = a.constrained && !xdeg && (x + g.x0 == 0 || x + g.x0 == g.nxg - 1);
      if (xb) zmask = 0xFFFFFFFFu;
    }
#pragma unroll
    for (int i = 0; i < G::LIT; ++i) {
      if (LTAIL && i == G::LIT - 1 && tid + i * NT >= G::LITEMS) break;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
          " cp.async.ca.shared.global [%0], [%1], 8, p;\n}\n" ::"r"(ldst[i] + buf * UBUF),
          "l"(base + loff[i]), "r"(zmask & (1u << i)) : "memory");
    }
    cp_async_commit();
  };

  // Z items: (q, yy, segment of ZS elements); lanes run along yy (odd pitch -> no bank conflicts)
  constexpr int ZSL = G::ZSLOTS;
  int zoff[ZSL], zeb[ZSL];
  unsigned zpart = 0u;  // balanced map: 2 bits per slot -- 0 whole item, 1 rows {0,1}, 2 rows {2,3}
#pragma unroll
  for (int i = 0; i < ZSL; ++i) {
    zeb[i] = TZE;  // inactive
    zoff[i] = 0;
    // item order: first rows 0..15 of every (q, segment) -- whole half-warps on one segment, so
    // the odd row pitch makes them conflict-free -- then the remaining rows, row-major across
    // (q, segment) (the mixed half-warps that remain are conflict-free for these pitches too)
    constexpr int R = NYin < 16 ? NYin : 16;
    constexpr int QS = Q * G::ZSEG;
    constexpr int T = QS * (NYin - R);
    int it = tid + i * NT;  // position in the item order; -1: none
    if constexpr (G::ZBAL) {
      // warps 0, 1 (no Y items): two whole head items; warps 2, 3: first halves of the other head
      // items; warps 4, 5: first halves of the tail items; warps 6, 7: the second halves of both
      const int w2 = tid >> 6, l = tid & 63;
      unsigned part = 0u;
      if (w2 == 0) it = l + 64 * i;
      else if (w2 == 1) { it = i == 0 ? 128 + l : -1; part = 1u; }
      else if (w2 == 2) { it = (i == 0 && l < T) ? QS * R + l : -1; part = 1u; }
      else { it = i == 0 ? 128 + l : (l < T ? QS * R + l : -1); part = 2u; }
      zpart |= part << (2 * i);
    }
    if (it >= 0 && it < G::ZITEMS) {
      int yy, qs;
      if (it < QS * R) {
        qs = it / R;
        yy = it - qs * R;
      } else {
        // rows past the first 16: the launcher's order (ztail_order), in which every 8 consecutive
        // lanes write 8 distinct 16-byte slots of the (A, B) buffer
        const int idx = T <= SPK_ZTAIL_MAX ? static_cast<int>(a.ztail[it - QS * R]) : it - QS * R;
        yy = R + idx / QS;
        qs = idx - (yy - R) * QS;
      }
      const int seg = qs % G::ZSEG, q = qs / G::ZSEG;
      if (!ydeg || yy == K) {
        zeb[i] = seg * G::ZS;
        zoff[i] = q * NYin + yy;  // row index
      }
    }
  }
  int zu[BULK ? ZSL : 1];  // TMA layout: offset of the item's box row in a plane buffer
  unsigned zq = 0u;           // ... and its stage (2 bits per item: virtual x-split boundary planes)
  unsigned zfl = 0u;          // ... and its boundary masks (5 bits per item)
  if constexpr (BULK) {
#pragma unroll
    for (int i = 0; i < ZSL; ++i) {
      const int q = zoff[i] / NYin, yy = zoff[i] - q * NYin;
      const long long e0 = (long long)q * a.su + (long long)(y_lo - K + yy) * g.nz + (z_lo - K);
      const uintptr_t addr = reinterpret_cast<uintptr_t>(u + e0);
      bpar0 |= static_cast<unsigned>((addr >> 3) & 1u) << i;
      zu[i] = (q * 2 + (yy & 1)) * G::REG + (yy >> 1) * G::W;
      zq |= static_cast<unsigned>(q) << (2 * i);
      // constrained operator on a tile next to the boundary: the boxes hold the raw boundary values,
      // which the operator treats as zero -- a boundary ROW zeroes its Z outputs, a boundary NODE
      // at the low / high end of the loaded z range is dropped from its element
      if (a.constrained && zeb[i] < TZE) {
        const int gy = y_lo - K + yy;
        if (gy == 0 || gy == g.ny - 1) zfl |= 1u << (5 * i);
        // (node z = 0 is the first loaded node of a tile one element in, or the first node of
        // element 0 = the left-element node 0 of an item that starts at element 1)
        if ((z_lo - K == 0 && zeb[i] == 0) || (ez0 == 0 && zeb[i] == 1)) zfl |= 2u << (5 * i);
        if (z_lo + TZ == g.nz - 1 && zeb[i] + G::ZS >= TZE) zfl |= 4u << (5 * i);
        if (ez0 == 0 && zeb[i] == 0) zfl |= 16u << (5 * i);  // node z = 0 is the first node of element 0
      }
    }
    static_assert(ZSL <= 6 && Q <= 4, "2 bits of stage, 5 mask bits per Z item");
  }
  // Y items: (q, z, segment of YS elements); lanes run along z
  int yoff[G::YIT], yeb[G::YIT];
#pragma unroll
  for (int i = 0; i < G::YIT; ++i) {
    // Y items are placed on the threads with the fewest Z items (balance inside the interval)
    constexpr int YOFF = (G::YITEMS % NT == 0) ? 0 : NT - (G::YITEMS % NT);
    const int it = (tid + NT - YOFF) % NT + i * NT;
    yeb[i] = TYE;
    yoff[i] = 0;
    if (it < G::YITEMS) {
      const int zl = it % TZ;
      const int rest = it / TZ;
      const int seg = rest % G::YSEG, q = rest / G::YSEG;
      if (zl < nzo) {
        yeb[i] = seg * G::YS;
        yoff[i] = q * 4096 + zl;  // packed (q, zl)
      }
    }
  }

  // ---------------- Z-phase: A = Mz u, B = Kz u ----------------
  auto zphase = [&](auto PB, int xp) {
    const int ub = parity_of(PB), ab = ub;
    const double* Ub = Us + ub * G::U_SZ;
    double2* AB = reinterpret_cast<double2*>(ABs + ab * 2 * G::AB_SZ);
    // constrained: the x-boundary planes are zero (the boxes hold the raw values: their Z outputs are
    // zeroed; virtual x-split: per stage)
    const bool vsp = BLOCK && a.vplanes != 0;
    const bool xzero = BULK && a.constrained && !vsp && (xp + g.x0 == 0 || xp + g.x0 == g.nxg - 1);
    const unsigned pflip = BULK ? ((static_cast<unsigned>(xp) & podd) ? ~0u : 0u) : 0u;
#pragma unroll
    for (int i = 0; i < ZSL; ++i) {
      if (zeb[i] >= nez) continue;
      const double* row = BULK ? Ub + zu[BULK ? i : 0] + (((bpar0 ^ pflip) >> i) & 1u) : Ub + zoff[i] * NZp;
      bool xz = xzero;
      if (BULK && vsp && a.constrained) {
        const int xgq = xp + g.x0 + static_cast<int>((zq >> (2 * i)) & 3u) * a.vplanes;
        xz = xgq == 0 || xgq == g.nxg - 1;
      }
      const unsigned fl = BULK ? (zfl >> (5 * i)) & 31u : 0u;
      if (BULK && (fl & 1u)) xz = true;
      double2* abrow = AB + zoff[i] * TZp;
      const int e_beg = zeb[i];
      if constexpr (G::ZBAL) {
        // balanced map: a whole item or half an element (warp-uniform per slot); ZS == 1
        const unsigned part = (zpart >> (2 * i)) & 3u;
        if (part != 0u) {
          constexpr int H = K / 2;
          const int e = e_beg, ez = ez0 + e;
          const double wl = ((FULL && !LOW) || ez > 0) ? 1.0 : 0.0, wr = (FULL || ez < g.Ez) ? 1.0 : 0.0;
          double L[K + 1], R[K + 1], oa[H], ob[H];
#pragma unroll
          for (int s = 0; s <= K; ++s) R[s] = row[K * e + K + s];
          if (BULK && (fl & 4u) && e == TZE - 1) R[K] = 0.0;
          if (BULK && (fl & 16u)) R[0] = 0.0;
          if (part == 1u && i == 0) {  // rows {0, 1}: the vertex row gathers the left element
#pragma unroll
            for (int s = 0; s < K; ++s) L[s] = row[K * e + s];
            L[K] = R[0];
            if (BULK && (fl & 2u)) L[0] = 0.0;
            elem2_half<K, true>(cf, L, R, wl, wr, oa, ob);
          } else {
            elem2_half<K, false>(cf, L, R, wl, wr, oa, ob);
          }
          if (BULK && xz) {
#pragma unroll
            for (int r = 0; r < H; ++r) oa[r] = ob[r] = 0.0;
          }
          const int zl0 = K * e + ((part == 1u && i == 0) ? 0 : H);
#pragma unroll
          for (int r = 0; r < H; ++r) abrow[zl0 + r] = make_double2(oa[r], ob[r]);
          continue;
        }
      }
      double L[K + 1], R[K + 1];
#pragma unroll
      for (int s = 0; s <= K; ++s) L[s] = row[K * e_beg + s];
      if (BULK && (fl & 2u)) L[0] = 0.0;
#pragma unroll
      for (int el = 0; el < G::ZS; ++el) {
        const int e = e_beg + el;
        if (e < nez) {
          R[0] = L[K];
#pragma unroll
          for (int s = 1; s <= K; ++s) R[s] = row[K * e + K + s];
          if (BULK && (fl & 4u) && e == TZE - 1) R[K] = 0.0;
          if (BULK && (fl & 16u) && el == 0) R[0] = 0.0;
          const int ez = ez0 + e;
          // (interior tiles may sit on the low boundary: element -1 does not exist, its slots hold
          // finite values of the neighbouring row or TMA zeros and get weight 0)
          const double wl = ((FULL && !LOW) || ez > 0) ? 1.0 : 0.0, wr = (FULL || ez < g.Ez) ? 1.0 : 0.0;
          double oa[K], ob[K];
          elem2<K>(cf, L, R, wl, wr, oa, ob);
          if (BULK && xz) {
#pragma unroll
            for (int r = 0; r < K; ++r) oa[r] = ob[r] = 0.0;
          }
#pragma unroll
          for (int r = 0; r < K; ++r) {
            const int zl = K * e + r;
            abrow[zl] = make_double2(oa[r], ob[r]);  // zl < TZ always; columns >= nzo are never read
          }
#pragma unroll
          for (int s = 0; s <= K; ++s) L[s] = R[s];
        }
      }
    }
  };

  // ---------------- Y-phase: MA = My A, C = Ky A + My B ----------------
  auto yphase = [&](auto PB, int mcbuf = -1) {
    const int ab = parity_of(PB), mc = mcbuf >= 0 ? mcbuf : ab;
    const double2* AB = reinterpret_cast<const double2*>(ABs + ab * 2 * G::AB_SZ);
    double2* MC = reinterpret_cast<double2*>(MCs + mc * 2 * G::MC_SZ);
    if (ydeg) {
      for (int it = tid; it < Q * TZ; it += NT) {
        const int q = it / TZ, zl = it - q * TZ;
        if (zl < nzo) MC[(q * TY) * TZp + zl] = AB[(q * NYin + K) * TZp + zl];
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < G::YIT; ++i) {
      if (yeb[i] >= ney) continue;
      const int q = yoff[i] >> 12, zl = yoff[i] & 4095;
      const double2* abcol = AB + (q * NYin) * TZp + zl;
      double2* mccol = MC + (q * TY) * TZp + zl;
      const int e_beg = yeb[i];
      double La[K + 1], Ra[K + 1], Lb[K + 1], Rb[K + 1];
#pragma unroll
      for (int s = 0; s <= K; ++s) {
        const double2 t = abcol[(K * e_beg + s) * TZp];
        La[s] = t.x;
        Lb[s] = t.y;
      }
#pragma unroll
      for (int el = 0; el < G::YS; ++el) {
        const int e = e_beg + el;
        if (e < ney) {
          Ra[0] = La[K];
          Rb[0] = Lb[K];
#pragma unroll
          for (int s = 1; s <= K; ++s) {
            const double2 t = abcol[(K * e + K + s) * TZp];
            Ra[s] = t.x;
            Rb[s] = t.y;
          }
          const int ey = ey0 + e;
          const double wl = ((FULL && !LOW) || ey > 0) ? 1.0 : 0.0, wr = (FULL || ey < g.Ey) ? 1.0 : 0.0;
          double om[K], oc[K];
          elem3<K>(cf, La, Ra, Lb, Rb, wl, wr, om, oc);
#pragma unroll
          for (int r = 0; r < K; ++r) {
            const int yl = K * e + r;  // yl < TY always; rows >= nyo are never read
            mccol[yl * TZp] = make_double2(om[r], oc[r]);
          }
#pragma unroll
          for (int s = 0; s <= K; ++s) { La[s] = Ra[s]; Lb[s] = Rb[s]; }
        }
      }
    }
  };

  // X-phase state
  double acc[PPT][Q][K + 1];
  int pyl[PPT], pzl[PPT], pyz[PPT];
  bool pv[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int p = tid + j * NT;
    pyl[j] = p / TZ;
    pzl[j] = p - pyl[j] * TZ;
    pyz[j] = (y_lo + pyl[j]) * g.nz + (z_lo + pzl[j]);
    pv[j] = (p < TY * TZ) && (FULL || (pyl[j] < nyo && pzl[j] < nzo));
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int s = 0; s <= K; ++s) acc[j][q][s] = 0.0;
  }
  double sumsq = 0.0;
  const bool dm_ident = a.dm_identity != 0;

  // ---------------- X-phase: stage mix + element-push accumulation ----------------
  // the plane's local index r within element ecur is uniform: dispatch to a copy with the x-table
  // column as compile-time register operands
  auto xphase_r = [&](auto RC, int x, auto MCP) {
    const int mc = parity_of(MCP);
    const double2* MC = reinterpret_cast<const double2*>(MCs + mc * 2 * G::MC_SZ);
    const int r_loc = parity_of(RC);  // compile-time for an IC<r>
    double cmx[K + 1], ckx[K + 1];
    if constexpr (std::is_same_v<decltype(RC), int>) {
      // one copy of the X-phase: the x-table column comes from constant memory by the (uniform)
      // plane index instead of five unrolled copies with register operands
#pragma unroll
      for (int s = 0; s <= K; ++s) {
        cmx[s] = c_hat[K - 1][0][r_loc][s];
        ckx[s] = c_hat[K - 1][1][r_loc][s];
      }
    } else {
#pragma unroll
      for (int s = 0; s <= K; ++s) {
        cmx[s] = cf.m(s, parity_of(RC));
        ckx[s] = cf.s(s, parity_of(RC));
      }
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (!pv[j]) continue;
      const int yl = pyl[j], zl = pzl[j];
      double ma[Q], cc[Q], pq[Q], qq[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double2 t = MC[(q * TY + yl) * TZp + zl];
        ma[q] = t.x;
        cc[q] = t.y;
      }
      if constexpr (BLOCK) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          pq[q] = fma(lamq[q], ma[q], a.tau * cc[q]);
          qq[q] = a.tau * ma[q];
        }
      } else {
        if (dm_ident) {  // D_M diagonal (the IRK operator I(x)M + tau A(x)K)
#pragma unroll
          for (int i = 0; i < Q; ++i) {
            double p = a.DM[i][i] * ma[i], s2 = 0.0;
#pragma unroll
            for (int jj = 0; jj < Q; ++jj) {
              p = fma(a.DK[i][jj], cc[jj], p);
              s2 = fma(a.DK[i][jj], ma[jj], s2);
            }
            pq[i] = p;
            qq[i] = s2;
          }
        } else {
#pragma unroll
          for (int i = 0; i < Q; ++i) {
            double p = 0.0, s2 = 0.0;
#pragma unroll
            for (int jj = 0; jj < Q; ++jj) {
              p = fma(a.DM[i][jj], ma[jj], p);
              p = fma(a.DK[i][jj], cc[jj], p);
              s2 = fma(a.DK[i][jj], ma[jj], s2);
            }
            pq[i] = p;
            qq[i] = s2;
          }
        }
      }
      const int y = y_lo + yl, z = z_lo + zl;
      if (xdeg) {
        epilogue<K, Q, BLOCK, EPI, FULL && !LOW>(a, b0, lamq, dtab, ith, 0, y, z, (long long)pyz[j], pq, sumsq);
        continue;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int s = 0; s <= K; ++s) acc[j][q][s] = fma(cmx[s], pq[q], fma(ckx[s], qq[q], acc[j][q][s]));
      if (r_loc == K) {
        // element ecur complete: nodes K*ecur + s, s < K
        if (ecur >= ex0) {
          // plain stores (CTA-uniform test): nothing of this element is a constrained identity row
          // -- unconstrained operator, or an interior tile away from the x = 0 plane -- so the
          // generic epilogue's per-node boundary tests and 64-bit index products are skipped
          bool fast = false;
          if constexpr (EPI == EPI_STORE && SPK_FAST_STORE)
            fast = !(BLOCK && a.vplanes != 0) &&
                   (!a.constrained || (FULL && !LOW && K * ecur + g.x0 != 0));
          if (fast) {
            double* vp = a.v + (BLOCK ? (long long)b0 * a.sv : 0) + (long long)(K * ecur) * plane_stride + pyz[j];
#pragma unroll
            for (int s = 0; s < K; ++s) {
#pragma unroll
              for (int q = 0; q < Q; ++q) __stcs(vp + q * a.sv, acc[j][q][s]);
              vp += plane_stride;
            }
          } else {
#pragma unroll
            for (int s = 0; s < K; ++s) {
              double val[Q];
#pragma unroll
              for (int q = 0; q < Q; ++q) val[q] = acc[j][q][s];
              const int xx = K * ecur + s;
              epilogue<K, Q, BLOCK, EPI, FULL && !LOW>(a, b0, lamq, dtab, ith, xx, y, z,
                                         (long long)xx * plane_stride + pyz[j], val, sumsq);
            }
          }
        }
        if (ecur + 1 == g.Ex && a.store_last) {  // final vertex plane nx-1 (left element only)
          double val[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) val[q] = acc[j][q][K];
          // virtual x-split: only the last range owns it (the others' is the next range's plane 0)
          epilogue<K, Q, BLOCK, EPI, FULL && !LOW>(a, b0, lamq, dtab, ith, K * g.Ex, y, z,
                                     (long long)(K * g.Ex) * plane_stride + pyz[j], val, sumsq,
                                     (BLOCK && a.vplanes) ? Q - 1 : 0);
        }
        // carry the shared vertex and start the next element with this plane as its local 0
        // (virtual x-split: the first range's halo element lies outside the domain -> no carry)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const bool ghost = BLOCK && a.vplanes && ecur + g.x0 / K + q * (a.vplanes / K) < 0;
          const double carry = ghost ? 0.0 : acc[j][q][K];
#pragma unroll
          for (int s = 0; s <= K; ++s) acc[j][q][s] = fma(cf.m(s, 0), pq[q], cf.s(s, 0) * qq[q]);
          acc[j][q][0] += carry;
        }
      }
    }
    if (!xdeg && r_loc == K) ++ecur;
  };
  auto xphase = [&](int x, auto mc) {
    const int r_loc = xdeg ? 0 : x - K * ecur;   // 0..K
    if constexpr (SPK_XR_RUNTIME) {
      xphase_r(r_loc, x, mc);
      return;
    }
    switch (r_loc) {
      case 0: xphase_r(IC<0>{}, x, mc); break;
      case 1: xphase_r(IC<1>{}, x, mc); break;
      case 2: if constexpr (K >= 2) xphase_r(IC<2>{}, x, mc); break;
      case 3: if constexpr (K >= 3) xphase_r(IC<3>{}, x, mc); break;
      case 4: if constexpr (K >= 4) xphase_r(IC<4>{}, x, mc); break;
    }
  };

  // Three-stage software pipeline, ONE barrier per plane: interval t runs Z(t), Y(t-1), X(t-2) on
  // disjoint double buffers (U/AB/MC indexed by plane parity) while U(t+1) is in flight. The loop is
  // unrolled by two so every buffer address is a compile-time offset.
  // split barrier: interval t waits for interval t-1's arrivals; MA/C plane t lives in buffer t % 3
  auto interval_split = [&](auto P, int t) {
    const auto p = P;  // == t & 1: a compile-time IC<p> (loop unrolled by two) or a runtime int
    const auto p1 = other_parity(P);
    if (t >= 1) mbar_wait(ibar, static_cast<unsigned>(t - 1) & 1u);
    if constexpr (BULK) {
      if (t < nplanes) mbar_wait(&ubar[parity_of(p)], static_cast<unsigned>(t >> 1) & 1u);
    }
    if (t + 1 < nplanes) load_plane(xs + t + 1, p1);
    if (t < nplanes) zphase(p, xs + t);
    if (t >= 1 && t - 1 < nplanes) yphase(p1, (t - 1) % 3);
    cp_async_wait_all();  // this thread's part of plane t+1 has landed
    if constexpr (SPK_WARP_ARRIVE) {
      // one arrival per warp: every arrival wakes the threads sleeping in the barrier wait
      // (NANOSLEEP.SYNCS), so 8 arrivals per phase cost the waiters fewer polls than 256
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(ibar);
    } else {
      mbar_arrive(ibar);
    }
    if (t >= 2) xphase(xs + t - 2, (t - 2) % 3);
  };
  auto interval = [&](auto P, int t) {
    constexpr int p = decltype(P)::value;  // == t & 1
    if constexpr (BULK) {
      if (t < nplanes) mbar_wait(&ubar[p], static_cast<unsigned>(t >> 1) & 1u);
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    if (t + 1 < nplanes) load_plane(xs + t + 1, IC<1 - p>{});
    if (t < nplanes) zphase(IC<p>{}, xs + t);
    if (t >= 1 && t - 1 < nplanes) yphase(IC<1 - p>{});
    if (t >= 2) xphase(xs + t - 2, IC<p>{});
  };
  if constexpr (BULK) {
    if (tid == 0) {
      mbar_init(&ubar[0], 1);
      mbar_init(&ubar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  spk_pdl_wait();  // everything above reads parameters / constants only
  load_plane(xs, IC<0>{});
  // unroll the plane loop by two (compile-time buffer offsets); measured on B200 to help every
  // instantiation except the stage-coupled k=2, Q=4 mix (C4's GMRES operator), whose doubled code
  // is slower (623 vs 575 us)
  constexpr bool UNROLL2 = BLOCK || !(K == 2 && Q == 4);
  if constexpr (G::SPLIT) {
    if (tid == 0) {
      mbar_init(ibar, SPK_WARP_ARRIVE ? NT / 32 : NT);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cp_async_wait_all();
    __syncthreads();  // plane 0 in shared memory, barrier initialised
    if constexpr (SPK_SPLIT_UNROLL2) {
      for (int t = 0; t < nplanes + 2; t += 2) {
        interval_split(IC<0>{}, t);
        if (t + 1 < nplanes + 2) interval_split(IC<1>{}, t + 1);
      }
    } else {  // one copy of the interval (half the hot loop's instruction footprint)
      for (int t = 0; t < nplanes + 2; ++t) interval_split(t & 1, t);
    }
    __syncthreads();
  } else if constexpr (UNROLL2) {
    for (int t = 0; t < nplanes + 2; t += 2) {
      interval(IC<0>{}, t);
      if (t + 1 < nplanes + 2) interval(IC<1>{}, t + 1);
    }
  } else {  // one copy of the interval with runtime buffer parity (smaller code)
    for (int t = 0; t < nplanes + 2; ++t) {
      const int p = t & 1;
      if constexpr (BULK) {
        if (t < nplanes) mbar_wait(&ubar[p], static_cast<unsigned>(t >> 1) & 1u);
      } else {
        cp_async_wait_all();
      }
      __syncthreads();
      if (t + 1 < nplanes) load_plane(xs + t + 1, 1 - p);
      if (t < nplanes) zphase(p, xs + t);
      if (t >= 1 && t - 1 < nplanes) yphase(1 - p);
      if (t >= 2) xphase(xs + t - 2, p);
    }
  }

  spk_pdl_trigger();  // after the plane pipeline: dependents launch during this grid's tail
  if constexpr (EPI == EPI_DINV) {
    // deterministic per-CTA partial: fixed-shape tree in shared memory
    __syncthreads();
    double* red = smem;
    red[tid] = sumsq;
    __syncthreads();
    for (int off = NT / 2; off > 0; off >>= 1) {
      if (tid < off) red[tid] += red[tid + off];
      __syncthreads();
    }
    if (tid == 0) {
      const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      a.partial[cta] = red[0];
    }
  }
}

#ifndef SPK_FULL_TILES
#define SPK_FULL_TILES 1
#endif

template <int K, int Q, bool BLOCK, int EPI>
__global__ void __launch_bounds__(Geo<K, Q>::NT,
                                  // (block mode only, and not the fused Chebyshev epilogue, which spills at
                                  // 64 registers; the pair mode's 2x2 epilogues lose at four CTAs:
                                  // measured C5-gmg 75.8 -> 84.2 ms / step)
                                  (Geo<K, Q>::MINB4_OK && BLOCK && EPI != EPI_CHEB) ? 4 : Geo<K, Q>::MINB)
    stage_apply_kernel(const __grid_constant__ SpkApplyArgs a, const __grid_constant__ SpkWsMaps maps) {
  extern __shared__ __align__(128) double smem[];
  using G = Geo<K, Q>;
  if constexpr (SPK_FULL_TILES) {
    // the loaded rows are y in [K (ey0 - 1), K (ey0 + TYE)] (same for z): inside the domain, every
    // element of the tile real (ey0 >= 1, ey0 + TYE <= Ey), and away from the constrained boundary
    const SpkDims& g = a.g;
    const int ez0 = blockIdx.x * G::TZE, ey0 = blockIdx.y * G::TYE;
    // (TMA boxes may read one double past the tile's last loaded node: still inside the array, an
    // interior tile never holds the array's last row; without tensor maps every tile takes the
    // generic body)
    // (constrained: with the TMA boxes a tile next to the boundary masks the loaded boundary row /
    // node in its Z sweep, so it is still an interior tile)
    const bool tma = SPK_TMA_LOAD && maps.bias >= 0;
    // (low boundary: rows below the plane are TMA zeros, the missing element gets weight 0 in the
    // Z / Y sweeps; only the ragged tiles on the high side take the generic body)
    const int lo = tma ? 0 : (a.constrained ? 2 : 1), hi = (a.constrained && !tma) ? 1 : 0;
    const bool full = g.Ey > 0 && g.Ez > 0 && g.Ex > 0 && ey0 >= lo && ez0 >= lo && ey0 + G::TYE + hi <= g.Ey &&
                      ez0 + G::TZE + hi <= g.Ez && (!SPK_TMA_LOAD || maps.bias >= 0);
    if (full) {
      if (ey0 == 0 || ez0 == 0) stage_apply_body<K, Q, BLOCK, EPI, 2>(a, maps, smem);
      else stage_apply_body<K, Q, BLOCK, EPI, 1>(a, maps, smem);
      return;
    }
  }
  stage_apply_body<K, Q, BLOCK, EPI, 0>(a, maps, smem);
}


// ---- small levels: direct banded gather, one thread per node -------------------------------------
// The sliding window pays its plane pipeline (cp.async latency + one barrier per plane) even when a
// level has a few hundred nodes: ~20-30 us per launch on the coarse levels of every V-cycle. There a
// thread per node gathers its (2K+1)^3 neighbourhood through L1 with the assembled 1D band rows (the
// same reference-element tables and scaled shifts as K1) and runs K1's epilogue unchanged.
#ifndef SPK_SMALL_WORK
#define SPK_SMALL_WORK SPK_SMALL_WORK_HOST   // n * (2K+1)^3 below which block-mode launches take this path
#endif
template <int K>
struct Band {
  // assembled 1D row of node class c (0 interior vertex, 1..K-1 element interior r, K first
  // boundary vertex, K+1 last boundary vertex) at offset d in [-K, K]
  static constexpr int NC = K + 2, W = 2 * K + 1;
  __device__ static void build(double* m, double* k) {  // [NC][W] each
    for (int idx = threadIdx.x; idx < NC * W; idx += blockDim.x) {
      const int c = idx / W, d = idx % W - K;
      double mv = 0.0, kv = 0.0;
      auto add = [&](int i_loc, int j_loc) {
        if (j_loc >= 0 && j_loc <= K) { mv += Hat<K>::M(i_loc, j_loc); kv += Hat<K>::S(i_loc, j_loc); }
      };
      if (c >= 1 && c < K) add(c, c + d);  // one element, local row c
      else {
        if (c != K) add(K, K + d);         // left element (absent at the first vertex)
        if (c != K + 1) add(0, d);         // right element (absent at the last vertex)
      }
      m[idx] = mv;
      k[idx] = kv;
    }
  }
  __device__ static int cls(int i, int n) {
    const int r = i % K;
    if (r != 0) return r;
    return i == 0 ? K : (i == n - 1 ? K + 1 : 0);
  }
};

// STAGED: the CTA first copies the x-planes its 256 nodes touch ([x_first - K, x_last + K]) into
// shared memory with coalesced loads -- one memory latency -- and gathers from there (the direct
// version waits out one L2 round trip per neighbour plane: 2K+1 of them)
template <int K, int EPI, bool STAGED>
__global__ void __launch_bounds__(256) small_apply_kernel(const __grid_constant__ SpkApplyArgs a) {
  // one CTA row per block (blockIdx.y), one thread per node; the epilogue is K1's with Q = 1
  using G = Geo<K, 1>;
  using BD = Band<K>;
  constexpr int W = BD::W;
  __shared__ double dtab[G::DT_SZ];
  __shared__ double bm[BD::NC * W], bk[BD::NC * W];
  __shared__ double red[256];
  extern __shared__ double ustage[];
  const int tid = threadIdx.x;
  const SpkDims g = a.g;
  const int b0 = a.blk_base + (int)blockIdx.y;
  const long long plane_n = (long long)g.ny * g.nz;
  int p0 = 0;
  double lamq[1], ith[1];
  lamq[0] = a.lam_uniform ? a.lam[0] : a.lam[b0 - a.blk_base];
  ith[0] = 1.0 / a.c2[b0 - a.blk_base];
  if constexpr (EPI != EPI_STORE) {
    constexpr int K1 = K + 1;
    for (int idx = tid; idx < K1 * K1 * K1; idx += blockDim.x) {
      const int cx = idx / (K1 * K1), cy = (idx / K1) % K1, cz = idx % K1;
      double mx, kx, my, ky, mz, kz;
      class_diag1<K>(cx, g.Ex, mx, kx);
      class_diag1<K>(cy, g.Ey, my, ky);
      class_diag1<K>(cz, g.Ez, mz, kz);
      const double dm = (mx * my) * mz;
      const double dk = ((kx * my) * mz + (mx * ky) * mz) + (mx * my) * kz;
      dtab[idx * G::DT_STRIDE] = 1.0 / (lamq[0] * dm + a.tau * dk);
    }
  }
  BD::build(bm, bk);
  spk_pdl_wait();  // the tables above need parameters only (they overlap the previous kernel)
  spk_pdl_trigger();
  if constexpr (STAGED) {
    const long long i0 = (long long)blockIdx.x * blockDim.x;
    const long long il = min(i0 + (long long)blockDim.x - 1, g.n - 1);
    p0 = max((int)(i0 / plane_n) - K, 0);
    const int p1 = min((int)(il / plane_n) + K, g.nx - 1);
    const double* src = a.u + (long long)b0 * a.su + (long long)p0 * plane_n;
    const long long cnt = (long long)(p1 - p0 + 1) * plane_n;
    for (long long j = tid; j < cnt; j += blockDim.x) ustage[j] = __ldg(src + j);
  }
  __syncthreads();
  double sumsq = 0.0;
  const long long i = (long long)blockIdx.x * blockDim.x + tid;
  if (i < g.n) {
    const int z = (int)(i % g.nz);
    const long long t = i / g.nz;
    const int y = (int)(t % g.ny), x = (int)(t / g.ny);
    const int cm = a.constrained ? 1 : 0;
    // per-axis band rows with out-of-range / masked (constrained boundary) neighbours zeroed, and
    // clamped (always valid) neighbour indices: fixed trip counts, independent loads
    double mzr[W], kzr[W], myr[W], kyr[W];
    int zi[W], yi[W];
    auto axis = [&](int c, int n, int E, double (&mr)[W], double (&kr)[W], int (&ix)[W]) {
      const int cl = E == 0 ? 0 : BD::cls(c, n);
#pragma unroll
      for (int d = 0; d < W; ++d) {
        const int j = c + d - K;
        const bool ok = E == 0 ? (d == K) : (j >= cm && j <= n - 1 - cm);
        mr[d] = ok ? (E == 0 ? 1.0 : bm[cl * W + d]) : 0.0;
        kr[d] = ok ? (E == 0 ? 0.0 : bk[cl * W + d]) : 0.0;
        ix[d] = min(max(j, 0), n - 1);
      }
    };
    axis(z, g.nz, g.Ez, mzr, kzr, zi);
    axis(y, g.ny, g.Ey, myr, kyr, yi);
    const double* u = STAGED ? ustage - (long long)p0 * plane_n : a.u + (long long)b0 * a.su;
    double v = 0.0;
    const int clx = g.Ex == 0 ? 0 : BD::cls(x, g.nx);
    for (int dxi = 0; dxi < W; ++dxi) {
      const int xx = x + dxi - K;
      const bool okx = g.Ex == 0 ? (dxi == K) : (xx >= cm && xx <= g.nx - 1 - cm);
      if (!okx) continue;
      const double mxv = g.Ex == 0 ? 1.0 : bm[clx * W + dxi], kxv = g.Ex == 0 ? 0.0 : bk[clx * W + dxi];
      if (mxv == 0.0 && kxv == 0.0) continue;
      const double* plane = u + (long long)xx * g.ny * g.nz;
      double A = 0.0, B = 0.0, C = 0.0;
#pragma unroll
      for (int dy = 0; dy < W; ++dy) {
        const double* line = plane + (long long)yi[dy] * g.nz;
        double uv[W];
#pragma unroll
        for (int dz = 0; dz < W; ++dz) uv[dz] = STAGED ? line[zi[dz]] : __ldg(line + zi[dz]);
        double am = 0.0, ak = 0.0;
#pragma unroll
        for (int dz = 0; dz < W; ++dz) {
          am = fma(mzr[dz], uv[dz], am);
          ak = fma(kzr[dz], uv[dz], ak);
        }
        A = fma(myr[dy], am, A);
        B = fma(kyr[dy], am, B);
        C = fma(myr[dy], ak, C);
      }
      v = fma(mxv, fma(lamq[0], A, a.tau * (B + C)), v);
      v = fma(a.tau * kxv, A, v);
    }
    double val[1] = {v};
    epilogue<K, 1, true, EPI>(a, b0, lamq, dtab, ith, x, y, z, i, val, sumsq);
  }
  if constexpr (EPI == EPI_DINV) {
    red[tid] = sumsq;
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
      if (tid < off) red[tid] += red[tid + off];
      __syncthreads();
    }
    if (tid == 0) a.partial[(long long)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
  }
}

}  // namespace
#include "stage_apply_ws.cuh"
namespace {

// K1w (stage_apply_ws.cuh), the warp-specialised variant, is a measured alternative and off by
// default (profiles/r02_k1w_*: C2 432 vs 399 us): SPK_WS=1 routes 3D launches on levels with at
// least SPK_WS_MIN nodes per axis to it
inline int spk_ws_min_nodes() {
  static int v = -2;
  if (v == -2) {
    const char* e = std::getenv("SPK_WS");
    if (!e || e[0] != '1') v = -1;
    else {
      const char* m = std::getenv("SPK_WS_MIN");
      v = m ? std::atoi(m) : 0;
    }
  }
  return v;
}

// Host: order of K1's Z-phase tail items (rows >= 16 of every (stage, segment)) such that each group
// of 8 consecutive items writes 8 distinct 16-byte slots (slot = (row * TZp + zl) mod 8 in double2
// units) -- greedy, once per geometry. Passed in the kernel parameters (computing it per thread at
// CTA setup cost more than it saved: profiles/r02_k1_ab.txt).
template <int K, int Q>
const unsigned char* ztail_order() {
  using G = Geo<K, Q>;
  constexpr int R = G::NYin < 16 ? G::NYin : 16;
  constexpr int QS = Q * G::ZSEG;
  constexpr int T = QS * (G::NYin - R);
  static unsigned char tab[SPK_ZTAIL_MAX] = {};
  static bool done = false;
  if (done || T <= 0 || T > SPK_ZTAIL_MAX) return tab;
  bool used[SPK_ZTAIL_MAX] = {};
  int pos = 0;
  while (pos < T) {
    unsigned slots = 0u;
    int got = 0;
    for (int c = 0; c < T && got < 8; ++c) {
      if (used[c]) continue;
      const int yy = R + c / QS, qs = c % QS, q = qs / G::ZSEG, seg = qs % G::ZSEG;
      const int sl = ((q * G::NYin + yy) * G::TZp + K * seg * G::ZS) & 7;
      if ((slots >> sl) & 1u) continue;
      slots |= 1u << sl;
      used[c] = true;
      tab[pos++] = static_cast<unsigned char>(c);
      ++got;
    }
    for (int c = 0; c < T && got < 8; ++c)
      if (!used[c]) {
        used[c] = true;
        tab[pos++] = static_cast<unsigned char>(c);
        ++got;
      }
  }
  done = true;
  return tab;
}

// SPK_CHUNK_MODEL=0: keep the host's fixed-target chunk count
inline bool spk_chunk_model() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("SPK_CHUNK_MODEL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}

template <int K, int Q, bool BLOCK, int EPI>
cudaError_t launch_one(const SpkApplyArgs& a_in, cudaStream_t s, int* nctas_out) {
  using G = Geo<K, Q>;
  SpkApplyArgs a = a_in;
  std::memcpy(a.ztail, ztail_order<K, Q>(), SPK_ZTAIL_MAX);
  constexpr long long W3 = (2 * K + 1) * (2 * K + 1) * (2 * K + 1);
  if constexpr (BLOCK) {
    // small whole-mesh levels: direct gather kernel (no plane pipeline)
    // (3D only: with a degenerate x axis the sliding window is a single plane and already cheap;
    // k <= 3: at k = 4 the 729-point gather loses to the window, measured)
    if (K <= 3 && a.vplanes == 0 && a.g.x0 == 0 && a.g.Ex > 0 && a.ex_begin == 0 && a.ex_end == a.g.Ex &&
        a.store_last && a.g.n * W3 <= (long long)SPK_SMALL_WORK) {
      dim3 grid((unsigned)((a.g.n + 255) / 256), (unsigned)a.nblk);
      if (nctas_out) *nctas_out = (int)(grid.x * grid.y);
      // staged x-planes: a run of 256 nodes touches at most 255/plane + 2 planes, plus K on each side
      const long long plane = (long long)a.g.ny * a.g.nz;
      const long long planes = std::min<long long>(a.g.nx, 255 / plane + 2 + 2 * K);
      const size_t stage_bytes = (size_t)(planes * plane) * sizeof(double);
      constexpr size_t STAGE_MAX = 160 * 1024;
      if (stage_bytes <= STAGE_MAX) {
        static bool configured_s = false;
        if (!configured_s) {
          cudaError_t e = cudaFuncSetAttribute(small_apply_kernel<K, EPI, true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)STAGE_MAX);
          if (e != cudaSuccess) return e;
          configured_s = true;
        }
        return spk_launch(small_apply_kernel<K, EPI, true>, grid, dim3(256), stage_bytes, s, a);
      }
      return spk_launch(small_apply_kernel<K, EPI, false>, grid, dim3(256), 0, s, a);
    }
  }
  SpkWsMaps maps;
  const bool have_maps = SPK_TMA_LOAD && ws_maps<K, Q>(a, BLOCK, &maps);
  if (!have_maps) maps.bias = -1;
  if constexpr (EPI != EPI_DINV) {
    const int wsmin = spk_ws_min_nodes();
    if (have_maps && wsmin >= 0 && a.g.nz >= wsmin && a.vplanes == 0)
      return launch_ws<K, Q, BLOCK, EPI>(a, maps, s, nctas_out);
  }
  const size_t smem = sizeof(double) * G::SMEM_DOUBLES;
  static bool configured = false;
  auto kern = stage_apply_kernel<K, Q, BLOCK, EPI>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int gz = (a.g.Ez + 1 + G::TZE - 1) / G::TZE;
  const int gy = a.g.Ey == 0 ? 1 : (a.g.Ey + 1 + G::TYE - 1) / G::TYE;
  const int nb = BLOCK ? a.nblk / Q : 1;  // CTA groups of Q blocks
  // x-chunk count by a makespan model over the instantiation's resident CTA slots: rounds of CTAs x
  // plane intervals per CTA (chunk planes + halo element + pipeline fill). The fixed "four waves of
  // 148" target ran C5's k = 3 operator (169 tiles) as 676 CTAs = 2.3 waves on 296 slots: 249 us
  // against 213 us with five chunks (2.85 waves); k = 4 / k = 2 at 289 tiles are flat in the count.
  static int slots = -1;
  if (slots < 0) {
    int occ = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::NT, smem) != cudaSuccess) occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    slots = occ * sms;
  }
  if (a.chunk_auto && a.g.Ex > 0 && slots > 0 && spk_chunk_model()) {
    const long long tiles = (long long)gz * gy * nb;
    const int nel = a.ex_end - a.ex_begin;
    // (large levels keep at least ~two rounds: the tiles are not uniform -- boundary tiles run the
    // generic body, the last tile row / column is thin -- and a single round of long CTAs measured
    // worse than two or three: C2 constrained 402 -> 450 us)
    const bool big = tiles * (nel / 4) >= 2LL * slots;
    long long best = -1;
    int best_xe = a.xe_chunk;
    for (int nch = 1; nch <= nel && nch <= 64; ++nch) {
      const int xe = (nel + nch - 1) / nch;
      if (xe < 2 && nel >= 2) break;
      const int n2 = (nel + xe - 1) / xe;
      if (big && tiles * n2 * 20 < 38LL * slots) continue;
      const long long rounds = (tiles * n2 + slots - 1) / slots;
      const long long cost = rounds * ((long long)xe * K + K + 3);
      if (best < 0 || cost < best) { best = cost; best_xe = xe; }
    }
    a.xe_chunk = best_xe;
    a.nchunks = (nel + best_xe - 1) / best_xe;
  }
  // the plane loads address a CTA's Q stage rows with 32-bit byte offsets from its first row
  if (((long long)(Q - 1) * a.su + a.g.n) * 8 > 0xFFFFFFFFLL) return cudaErrorInvalidValue;
  dim3 grid(gz, gy, a.nchunks * nb);
  if (nctas_out) *nctas_out = gz * gy * a.nchunks * nb;
  return spk_launch(kern, grid, dim3(G::NT), smem, s, a, maps);
}

#define SPK_EPIS(K, Q, B)                                                   \
  switch (epi) {                                                            \
    case EPI_STORE: return launch_one<K, Q, B, EPI_STORE>(a, s, n);         \
    case EPI_RESID: return launch_one<K, Q, B, EPI_RESID>(a, s, n);         \
    case EPI_CHEB: return launch_one<K, Q, B, EPI_CHEB>(a, s, n);           \
    case EPI_DINV: return launch_one<K, Q, B, EPI_DINV>(a, s, n);           \
  }                                                                         \
  return cudaErrorInvalidValue;

template <int K>
cudaError_t dispatch_k(int Q, bool block_mode, int epi, const SpkApplyArgs& a, cudaStream_t s, int* n) {
  if (block_mode) {  // Q = blocks per CTA (diagonal mix, per-block shifts)
    switch (Q) {
      case 1: SPK_EPIS(K, 1, true)
      case 2: SPK_EPIS(K, 2, true)
      case 3: SPK_EPIS(K, 3, true)
      case 4: SPK_EPIS(K, 4, true)
    }
    return cudaErrorInvalidValue;
  }
  switch (Q) {
    case 1: return launch_one<K, 1, false, EPI_STORE>(a, s, n);
    case 2: SPK_EPIS(K, 2, false)
    case 3: return launch_one<K, 3, false, EPI_STORE>(a, s, n);
    case 4: return launch_one<K, 4, false, EPI_STORE>(a, s, n);
  }
  return cudaErrorInvalidValue;
}
#undef SPK_EPIS

}  // namespace
