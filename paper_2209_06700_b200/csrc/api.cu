// C-ABI host layer of libspk: discretisation setup (Q_k element tables on GLL nodes, transfer
// tables, per-level dims) and stream-ordered kernel launches. See include/spk.h for the contract.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/spk.h"
#include "spk_internal.cuh"
#include "spk_vecops.cuh"

namespace {
// NVTX range per C-ABI entry point (free when no profiler is attached): the timeline of a step
// (ncu / nsight) shows which reference operation each kernel serves
struct SpkRange {
  explicit SpkRange(const char* name) { nvtxRangePushA(name); }
  ~SpkRange() { nvtxRangePop(); }
};
}  // namespace
#define SPK_RANGE(name) SpkRange spk_range_guard_(name)

struct spk_ctx {
  int dim = 0, max_level = 0, K = 0;
  std::vector<SpkDims> dims;
  std::vector<SpkTab> tabs;
  std::vector<double> h;
  // per-level x-slab window (spk_ctx_set_slab): nodes of elements [ex_begin, ex_end) (+ the last
  // vertex plane if store_last) are produced; a whole-mesh level produces everything
  std::vector<int> ex_begin, ex_end, store_last;
  double xi[SPK_KMAX + 1];
  double P[(2 * SPK_KMAX + 1) * (SPK_KMAX + 1)];
  int target_ctas = 0;    // 0: automatic x-chunking
  int fill_wave = 1;      // automatic chunking may shorten chunks to fill one wave (SPK_FILL_WAVE=0: off)
  int fuse_transfer = 1;  // fused 3D prolongation on whole-mesh levels (SPK_FUSE_TRANSFER=0: three sweeps)
  int mgs_pair = 3;                  // paired MGS sweeps: bit 0 large vectors, bit 1 cooperative column (SPK_MGS_PAIR)
  int mgs_coop = 1;                  // cooperative single-launch MGS column for small vectors (SPK_MGS_COOP)
  long long mgs_coop_max = 1LL << 25; // ... up to this many doubles (measured: C5 -5 %, C4 at 68M neutral)
  long long cv_max_nodes = 2200;  // fused coarse V-cycle: top level up to this many nodes (SPK_CV_MAXN;
                                  // measured: a single CTA loses at 17^3 nodes, k=2 C3 V-cycle 479 vs 569 us)
  long long fuse_restrict_max = 1LL << 22;  // fused 3D restriction up to nblk * n fine DoFs (SPK_FUSE_RESTRICT_MAX)
  // block-DoFs from which Chebyshev steps run split; launches of >= 3 blocks always run split (their
  // fused CHEB variants spill at 128 registers). Measured: C1 (2 blocks, tiny levels) prefers fused,
  // C3 / C4 (3-4 blocks) split on every level, single-block V-cycles split from ~2^18 DoFs.
  long long split_cheb_min = 1LL << 18;
  int split_cheb_nblk = 3;  // (SPK_CHEB_SPLIT_NBLK)
  int per_cta2_epi = 1;   // epilogues (bit mask over SpkEpi) that take the two-per-CTA launch (SPK_PER_CTA2_EPI)
  int vsplit_v = 0;       // virtual x-ranges per CTA of a single-block launch (SPK_VSPLIT_V: 4 or 2; 0: automatic)
  // blocks swept together by one K1 CTA (SPK_PER_CTA_MAX; 0: two per CTA where SPK_PER_CTA2_* allow.
  // Measured on C4: two per CTA wins the STORE launch alone, 531 -> 484 us, but not the step, 211 -> 220 ms)
  int per_cta_max = 4;
  long long per_cta2_min = 1LL << 16;  // ... two per CTA from this many nodes per block (SPK_PER_CTA2_MIN)
  int vsplit = 1;         // single-block K1 launches sweep 4 x-ranges per CTA (virtual x-split)
  // device scratch (lazily allocated on first device call)
  double* partial = nullptr;
  unsigned* counter = nullptr;
  int partial_cap = 0;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SPK_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---- 1D reference element on [0,1]: GLL nodes, Gauss rule, Lagrange basis ----
void gll_nodes(int K, double* xi) {
  // Gauss-Lobatto-Legendre points mapped to [0,1] (closed forms for K <= 4)
  switch (K) {
    case 1: xi[0] = 0.0; xi[1] = 1.0; break;
    case 2: xi[0] = 0.0; xi[1] = 0.5; xi[2] = 1.0; break;
    case 3: {
      const double a = std::sqrt(5.0) / 10.0;
      xi[0] = 0.0; xi[1] = 0.5 - a; xi[2] = 0.5 + a; xi[3] = 1.0;
      break;
    }
    case 4: {
      const double a = std::sqrt(21.0) / 14.0;
      xi[0] = 0.0; xi[1] = 0.5 - a; xi[2] = 0.5; xi[3] = 0.5 + a; xi[4] = 1.0;
      break;
    }
  }
}

void gauss_legendre01(int m, double* x, double* w) {
  // Newton on P_m, mapped to [0,1]
  for (int i = 0; i < m; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (m + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= m; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (m == 1) { p1 = z; p0 = 1.0; }
      const double dp = m * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= m; ++k) {
      const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    const double dp = (m == 1) ? 1.0 : m * (z * p1 - p0) / (z * z - 1.0);
    x[m - 1 - i] = 0.5 * (z + 1.0);
    w[m - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);  // weight on [0,1] = 2/((1-z^2)P'^2) / 2
  }
  if (m == 1) { x[0] = 0.5; w[0] = 1.0; }
}

double lagr(const double* xi, int K, int a, double x) {
  double v = 1.0;
  for (int m = 0; m <= K; ++m)
    if (m != a) v *= (x - xi[m]) / (xi[a] - xi[m]);
  return v;
}

double lagr_d(const double* xi, int K, int a, double x) {
  double s = 0.0;
  for (int m = 0; m <= K; ++m) {
    if (m == a) continue;
    double t = 1.0 / (xi[a] - xi[m]);
    for (int l = 0; l <= K; ++l)
      if (l != a && l != m) t *= (x - xi[l]) / (xi[a] - xi[l]);
    s += t;
  }
  return s;
}

SpkDims dims_of(const spk_ctx* c, int level) { return c->dims[level]; }

int check_level(const spk_ctx* c, int level) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  if (level < 0 || level > c->max_level)
    return fail(SPK_ECONFIG, "level " + std::to_string(level) + " outside hierarchy");
  return SPK_OK;
}

int ensure_scratch(spk_ctx* c, int need) {
  if (c->partial_cap >= need && c->counter) return SPK_OK;
  if (c->partial) {
    cudaFree(c->partial);
    c->partial = nullptr;  // never leave a dangling buffer behind a failed cudaMalloc below
    c->partial_cap = 0;
  }
  if (!c->counter) {
    cudaError_t e = cudaMalloc(&c->counter, 64 * sizeof(unsigned));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(counter)");
    e = cudaMemset(c->counter, 0, 64 * sizeof(unsigned));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(counter)");
  }
  int cap = need < (1 << 16) ? (1 << 16) : need;
  cudaError_t e = cudaMalloc(&c->partial, (size_t)cap * sizeof(double));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(partial)");
  c->partial_cap = cap;
  return SPK_OK;
}

// a level that is the whole mesh (no slab window)
bool whole_level(const spk_ctx* c, int level) {
  const SpkDims& g = c->dims[level];
  return g.x0 == 0 && c->ex_begin[level] == 0 && (c->ex_end[level] == 0 || c->ex_end[level] == g.Ex) &&
         c->store_last[level];
}

// whole-mesh 3D level that block-mode K1 launches run with the direct small-level kernel
// (stage_apply.cuh launch_one: k <= 3 and n (2k+1)^3 <= SPK_SMALL_WORK)
bool small_level(const spk_ctx* c, int level) {
  const SpkDims& g = c->dims[level];
  const long long w1 = 2LL * c->K + 1;
  return c->K <= 3 && c->dim == 3 && g.Ex > 0 && whole_level(c, level) &&
         g.n * w1 * w1 * w1 <= (long long)SPK_SMALL_WORK_HOST;
}

// x-chunking of the sliding window: enough CTAs to fill every SM about twice
void set_chunking(const spk_ctx* c, SpkApplyArgs& a, int K, int nb, int Qcta) {
  const int tye = spk_apply_geo(K, Qcta, 2), tze = spk_apply_geo(K, Qcta, 3);  // the kernel's (y,z) tile
  const int gz = (a.g.Ez + 1 + tze - 1) / tze;
  const int gy = a.g.Ey == 0 ? 1 : (a.g.Ey + 1 + tye - 1) / tye;
  const long long tiles = (long long)gz * gy * nb;
  if (a.g.Ex == 0) { a.nchunks = 1; a.xe_chunk = 1; a.ex_begin = 0; a.ex_end = 0; return; }
  if (a.ex_end <= a.ex_begin) { a.ex_begin = 0; a.ex_end = a.g.Ex; }
  const int nel = a.ex_end - a.ex_begin;
  // ~4 waves of one CTA per SM: fewer, longer x-chunks amortise the one-element chunk halo
  // (C2 is flat between 4 and 6 waves; C4's block-mode sweeps prefer 4, tools/prof_apply.py)
  // (virtual x-split launches: each chunk pays a halo element of a short virtual block, fewer chunks
  // measured better: C5 finest level STORE 125 -> 118 us, residual 133 -> 124 us with ~2.7 waves)
  const long long target = c->target_ctas > 0 ? c->target_ctas : (a.vplanes ? 400 : 4 * 148);
  long long nch = (target + tiles - 1) / tiles;
  if (nch < 1) nch = 1;
  if (nch > nel) nch = nel;
  // keep at least 4 elements per chunk (the chunk pays one halo element) ...
  while (nch > 1 && nel / nch < 4) --nch;
  // ... unless that leaves part of the GPU idle: on small and mid-size levels a launch is bound by
  // the plane-pipeline latency of one CTA, so shorter chunks (down to one element) that fill one wave
  // of two CTAs per SM finish sooner than a few long ones
  if (c->target_ctas <= 0 && c->fill_wave) {
    const long long wave = 2LL * 148;
    long long fill = wave / tiles;
    if (fill > nel) fill = nel;
    if (fill > nch) nch = fill;
  }
  a.xe_chunk = (int)((nel + nch - 1) / nch);
  a.nchunks = (nel + a.xe_chunk - 1) / a.xe_chunk;
  // automatic chunking of plain launches: the launcher refines the count with the instantiation's
  // resident-CTA slots (stage_apply.cuh rechunk)
  a.chunk_auto = (c->target_ctas <= 0 && a.vplanes == 0) ? 1 : 0;
}

SpkApplyArgs base_args(const spk_ctx* c, int level) {
  SpkApplyArgs a;
  std::memset(&a, 0, sizeof(a));
  a.g = c->dims[level];
  a.t = c->tabs[level];
  a.ex_begin = c->ex_begin[level];
  a.ex_end = c->ex_end[level];
  a.store_last = c->store_last[level];
  a.hd = std::pow(c->h[level], c->dim);
  a.hk = std::pow(c->h[level], c->dim - 2);
  return a;
}

int launch_apply(spk_ctx* c, int Q, bool block_mode, int epi, SpkApplyArgs& a0, cudaStream_t s,
                 int* nctas = nullptr) {
  // the kernels work with reference-element tables: M = h^d M_hat, K = h^(d-2) K_hat
  SpkApplyArgs a = a0;
  bool ident = !block_mode;
  for (int i = 0; i < SPK_QMAX; ++i)
    for (int j = 0; j < SPK_QMAX; ++j) {
      if (i < Q && j < Q && i != j && a0.DM[i][j] != 0.0) ident = false;
      a.DM[i][j] *= a0.hd;
      a.DK[i][j] *= a0.hk;
    }
  a.dm_identity = ident ? 1 : 0;  // D_M diagonal (e.g. I (x) M): Q fewer FMAs per stage-DoF
  set_chunking(c, a, c->K, block_mode ? a.nblk / Q : 1, Q);
  for (int i = 0; i < SPK_BMAX; ++i) a.lam[i] *= a0.hd;
  a.tau *= a0.hk;
  a.jre *= a0.hd;
  a.jim *= a0.hd;
  cudaError_t e = spk_launch_apply(c->K, Q, block_mode, epi, a, s, nctas);
  if (e != cudaSuccess) return cuda_fail(e, "stage_apply launch");
  return SPK_OK;
}

int apply_blocks_chunked(spk_ctx* c, int level, int nblk, const double* lams, int lam_uniform,
                         double tau, int constrained, int epi, SpkApplyArgs a, cudaStream_t s,
                         const double* c1s, const double* c2s) {
  // one block: a CTA of Q = 1 leaves most threads idle in the Z / Y phases; sweep V consecutive
  // x-ranges of the block as V "virtual blocks" instead (whole-mesh 3D levels with >= 8 elements)
  const SpkDims& g = a.g;
  // (not for the fused Chebyshev epilogue: its 4-stage variant spills at 128 registers)
  // (not on levels the direct small-level kernel takes: stage_apply.cuh launch_one)
  if (nblk == 1 && c->vsplit && !small_level(c, level) && epi != EPI_CHEB && c->dim == 3 && g.Ex >= 8 && g.x0 == 0 &&
      a.ex_begin == 0 && (a.ex_end == 0 || a.ex_end == g.Ex)) {
    // (degrees <= 3: two ranges per CTA at four CTAs per SM, stage_apply.cuh SPK_MINB4 -- measured C5
    // 95.1 -> 89.0 ms / step, C5-gmg 77.7 -> 74.6)
    const int vpref = c->vsplit_v > 0 ? c->vsplit_v : (c->K <= 3 ? 2 : 4);
    const int V = (g.Ex % 4 == 0 && vpref != 2) ? 4 : 2;
    const int Ev = g.Ex / V;
    const long long vs = (long long)c->K * Ev * g.ny * g.nz;
    SpkApplyArgs b = a;
    b.su = vs; b.sv = vs; b.se = vs;
    b.vplanes = c->K * Ev;
    b.g.Ex = Ev;
    b.g.nx = c->K * Ev + 1;
    b.g.n = (long long)b.g.nx * g.ny * g.nz;
    b.ex_begin = 0; b.ex_end = Ev;
    b.blk_base = 0; b.nblk = V;
    b.lam_uniform = 1; b.lam[0] = lams[0];
    b.tau = tau; b.constrained = constrained;
    for (int i = 0; i < V; ++i) {
      b.c1[i] = c1s ? c1s[0] : 0.0;
      b.c2[i] = c2s ? c2s[0] : 0.0;
    }
    return launch_apply(c, V, true, epi, b, s);
  }
  // launch in groups of at most SPK_BMAX blocks so per-block coefficients fit the parameter block;
  // inside a launch every CTA sweeps `per_cta` blocks together (1..4) to share the halo loads,
  // index math and barriers of the plane pipeline
  for (int b0 = 0; b0 < nblk;) {
    int nb = std::min(SPK_BMAX, nblk - b0);
    int per_cta = 1;
    // low degrees, large levels, an even number of blocks: two blocks per CTA at four CTAs per SM
    // (stage_apply.cuh SPK_MINB4) beat four per CTA at two
    int qmax = c->per_cta_max;
    if (qmax <= 0)
      qmax = (c->K <= 3 && nb % 2 == 0 && a.g.n >= c->per_cta2_min && ((c->per_cta2_epi >> epi) & 1)) ? 2 : 4;
    for (int q = qmax; q >= 2; --q)
      if (nb >= q) { per_cta = q; break; }
    nb = (nb / per_cta) * per_cta;
    a.blk_base = b0;
    a.nblk = nb;
    a.lam_uniform = lam_uniform;
    a.tau = tau;
    a.constrained = constrained;
    if (lam_uniform) a.lam[0] = lams[0];
    else
      for (int i = 0; i < nb; ++i) a.lam[i] = lams[b0 + i];
    for (int i = 0; i < nb && i < SPK_BMAX; ++i) {
      a.c1[i] = c1s ? c1s[b0 + i] : 0.0;
      a.c2[i] = c2s ? c2s[b0 + i] : 0.0;
    }
    // blocks are addressed as blk*su from the base pointer, so pass the unshifted base
    int rc = launch_apply(c, per_cta, true, epi, a, s);
    if (rc) return rc;
    b0 += nb;
  }
  return SPK_OK;
}

// row range (x*ny + y) of the produced planes of a level and the row-kernel geometry
SpkRowArgs row_args(const spk_ctx* c, int level) {
  SpkRowArgs a;
  std::memset(&a, 0, sizeof(a));
  a.g = c->dims[level];
  a.t = c->tabs[level];
  int xb = 0, xe = a.g.nx;
  if (a.g.Ex > 0) {
    xb = c->K * c->ex_begin[level];
    xe = c->K * c->ex_end[level] + ((c->store_last[level] && c->ex_end[level] == a.g.Ex) ? 1 : 0);
  }
  a.row0 = xb * a.g.ny;
  a.nrows = (xe - xb) * a.g.ny;
  int tpr = 1;
  while (tpr < a.g.nz && tpr < 128) tpr *= 2;
  a.tpr = tpr;
  a.constrained = 1;
  return a;
}

// the fused K1 Chebyshev epilogue is latency-bound on its global operands at large levels: there
// the step runs as a K1 STORE of w = A d followed by the pointwise update (more bytes, near the
// HBM roofline); small (L2-resident) levels keep the single fused launch (ctx->split_cheb_min)

bool cheb_split(const spk_ctx* c, int level, int nblk) {
  // levels the direct small-level kernel takes (one CTA row per block) always fuse: there a launch
  // costs more than the epilogue's loads
  if (small_level(c, level)) return false;
  return nblk >= c->split_cheb_nblk || (long long)nblk * c->dims[level].n >= c->split_cheb_min;
}

}  // namespace

bool spk_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("SPK_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

long long spk_pdl_max_ctas() {
  // measured: PDL pays on latency-bound launches (one wave) and costs on large grids (C4 V-cycle
  // +10 % with every launch of up to 8 CTAs per SM attributed)
  static long long m = -1;
  if (m < 0) {
    const char* e = std::getenv("SPK_PDL_MAX");
    m = e ? std::atoll(e) : 148;
  }
  return m;
}

extern "C" {

int spk_version(void) { return 1; }

const char* spk_last_error(void) { return g_err.c_str(); }

int spk_ctx_create(int dim, int max_level, int degree, spk_ctx** out) {
  if (!out) return fail(SPK_ECONFIG, "null output pointer");
  if (dim < 1 || dim > 3) return fail(SPK_ECONFIG, "dim must be 1, 2 or 3, got " + std::to_string(dim));
  if (degree < 1 || degree > SPK_KMAX)
    return fail(SPK_EUNSUPPORTED, "degree must be in [1, 4], got " + std::to_string(degree));
  if (max_level < 1 || max_level > 10)
    return fail(SPK_ECONFIG, "max_level must be in [1, 10], got " + std::to_string(max_level));
  spk_ctx* c = new spk_ctx();
  if (const char* e = std::getenv("SPK_CHEB_SPLIT")) c->split_cheb_min = std::atoll(e);  // tuning override
  if (const char* e = std::getenv("SPK_CHEB_SPLIT_NBLK")) c->split_cheb_nblk = std::atoi(e);
  if (const char* e = std::getenv("SPK_VSPLIT")) c->vsplit = std::atoi(e);
  if (const char* e = std::getenv("SPK_PER_CTA_MAX")) c->per_cta_max = std::max(0, std::min(4, std::atoi(e)));
  if (const char* e = std::getenv("SPK_PER_CTA2_EPI")) c->per_cta2_epi = std::atoi(e);
  if (const char* e = std::getenv("SPK_VSPLIT_V")) c->vsplit_v = std::atoi(e);
  if (const char* e = std::getenv("SPK_PER_CTA2_MIN")) c->per_cta2_min = std::atoll(e);
  if (const char* e = std::getenv("SPK_FILL_WAVE")) c->fill_wave = std::atoi(e);
  if (const char* e = std::getenv("SPK_FUSE_TRANSFER")) c->fuse_transfer = std::atoi(e);
  if (const char* e = std::getenv("SPK_FUSE_RESTRICT_MAX")) c->fuse_restrict_max = std::atoll(e);
  if (const char* e = std::getenv("SPK_CV_MAXN")) c->cv_max_nodes = std::atoll(e);
  if (const char* e = std::getenv("SPK_MGS_COOP")) c->mgs_coop = std::atoi(e);
  if (const char* e = std::getenv("SPK_MGS_PAIR")) c->mgs_pair = std::atoi(e);
  if (const char* e = std::getenv("SPK_MGS_COOP_MAX")) c->mgs_coop_max = std::atoll(e);
  c->dim = dim;
  c->max_level = max_level;
  c->K = degree;
  const int K = degree;
  gll_nodes(K, c->xi);
  // reference element matrices with the exact (K+1)-point Gauss rule
  double gx[SPK_KMAX + 1], gw[SPK_KMAX + 1];
  gauss_legendre01(K + 1, gx, gw);
  double Mh[SPK_KMAX + 1][SPK_KMAX + 1] = {}, Kh[SPK_KMAX + 1][SPK_KMAX + 1] = {};
  for (int a = 0; a <= K; ++a)
    for (int b = 0; b <= K; ++b) {
      double m = 0.0, k = 0.0;
      for (int q = 0; q <= K; ++q) {
        m += gw[q] * lagr(c->xi, K, a, gx[q]) * lagr(c->xi, K, b, gx[q]);
        k += gw[q] * lagr_d(c->xi, K, a, gx[q]) * lagr_d(c->xi, K, b, gx[q]);
      }
      Mh[a][b] = m;
      Kh[a][b] = k;
    }
  // symmetrise (exact symmetry of the element matrices)
  for (int a = 0; a <= K; ++a)
    for (int b = a + 1; b <= K; ++b) {
      Mh[b][a] = Mh[a][b];
      Kh[b][a] = Kh[a][b];
    }
  // prolongation table: fine local position f in [0, 2K] of a coarse element
  std::memset(c->P, 0, sizeof(c->P));
  for (int f = 0; f <= 2 * K; ++f) {
    const double pos = (f <= K) ? 0.5 * c->xi[f] : 0.5 + 0.5 * c->xi[f - K];
    for (int j = 0; j <= K; ++j) {
      double v = lagr(c->xi, K, j, pos);
      if (f == 0) v = (j == 0) ? 1.0 : 0.0;
      if (f == 2 * K) v = (j == K) ? 1.0 : 0.0;
      if (f == K && K % 2 == 0) v = (j == K / 2) ? 1.0 : 0.0;  // midpoint is a coarse node
      c->P[f * (SPK_KMAX + 1) + j] = v;
    }
  }
  for (int l = 0; l <= max_level; ++l) {
    const int N = 1 << l;
    const int nax = K * N + 1;
    SpkDims g;
    g.nz = nax; g.Ez = N;
    g.ny = dim >= 2 ? nax : 1; g.Ey = dim >= 2 ? N : 0;
    g.nx = dim >= 3 ? nax : 1; g.Ex = dim >= 3 ? N : 0;
    g.n = (long long)g.nx * g.ny * g.nz;
    g.x0 = 0; g.nxg = g.nx; g.Exg = g.Ex;
    const double h = 1.0 / N;
    SpkTab t;
    std::memset(&t, 0, sizeof(t));
    for (int a = 0; a <= K; ++a)
      for (int b = 0; b <= K; ++b) {
        t.Me[a][b] = h * Mh[a][b];
        t.Ke[a][b] = Kh[a][b] / h;
      }
    c->dims.push_back(g);
    c->tabs.push_back(t);
    c->h.push_back(h);
    c->ex_begin.push_back(0);
    c->ex_end.push_back(g.Ex);
    c->store_last.push_back(1);
  }
  *out = c;
  return SPK_OK;
}

int spk_ctx_destroy(spk_ctx* c) {
  if (!c) return SPK_OK;
  if (c->partial) cudaFree(c->partial);
  if (c->counter) cudaFree(c->counter);
  delete c;
  return SPK_OK;
}

int spk_ctx_set_slab(spk_ctx* c, int level, int x_elems, int x0_plane, int ex_begin, int ex_end,
                     int store_last) {
  if (int rc = check_level(c, level)) return rc;
  if (c->dim != 3) return fail(SPK_ECONFIG, "slab windows need a 3D hierarchy");
  SpkDims& g = c->dims[level];
  const int Eg = 1 << level;
  if (x_elems < 1 || ex_begin < 0 || ex_end > x_elems || ex_begin >= ex_end || x0_plane % c->K != 0 ||
      x0_plane / c->K + ex_begin < 0 || x0_plane / c->K + ex_end > Eg)
    return fail(SPK_ECONFIG, "bad slab window at level " + std::to_string(level));
  g.Ex = x_elems;
  g.nx = c->K * x_elems + 1;
  g.n = (long long)g.nx * g.ny * g.nz;
  g.x0 = x0_plane;
  g.Exg = Eg;
  g.nxg = c->K * Eg + 1;
  c->ex_begin[level] = ex_begin;
  c->ex_end[level] = ex_end;
  c->store_last[level] = store_last;
  return SPK_OK;
}

int spk_level_info(const spk_ctx* c, int level, int* n_per_axis, long long* n_dofs, double* h,
                   int* n_elems) {
  if (int rc = check_level(c, level)) return rc;
  const SpkDims& g = c->dims[level];
  if (n_per_axis) *n_per_axis = g.nz;
  if (n_dofs) *n_dofs = g.n;
  if (h) *h = c->h[level];
  if (n_elems) *n_elems = g.Ez;
  return SPK_OK;
}

int spk_level_tables(const spk_ctx* c, int level, double* Me, double* Ke) {
  if (int rc = check_level(c, level)) return rc;
  const int K = c->K;
  for (int a = 0; a <= K; ++a)
    for (int b = 0; b <= K; ++b) {
      if (Me) Me[a * (K + 1) + b] = c->tabs[level].Me[a][b];
      if (Ke) Ke[a * (K + 1) + b] = c->tabs[level].Ke[a][b];
    }
  return SPK_OK;
}

int spk_nodes_1d(const spk_ctx* c, int level, double* out) {
  if (int rc = check_level(c, level)) return rc;
  const int K = c->K, N = c->dims[level].Ez;
  const double h = c->h[level];
  for (int e = 0; e < N; ++e)
    for (int r = 0; r < K; ++r) out[K * e + r] = (e + c->xi[r]) * h;
  out[K * N] = 1.0;
  out[0] = 0.0;
  return SPK_OK;
}

int spk_prolong_table(const spk_ctx* c, double* P) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  const int K = c->K;
  for (int f = 0; f <= 2 * K; ++f)
    for (int j = 0; j <= K; ++j) P[f * (K + 1) + j] = c->P[f * (SPK_KMAX + 1) + j];
  return SPK_OK;
}

int spk_apply_smem(int degree, int Q) { return spk_apply_smem_bytes(degree, Q); }

int spk_set_chunks(spk_ctx* c, int target_ctas) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  c->target_ctas = target_ctas;
  return SPK_OK;
}

int spk_set_vsplit(spk_ctx* c, int on) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  c->vsplit = on;
  return SPK_OK;
}

int spk_set_cheb_split(spk_ctx* c, long long min_block_dofs) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  c->split_cheb_min = min_block_dofs;
  return SPK_OK;
}

int spk_stage_apply(spk_ctx* c, int level, int Q, const double* DM, const double* DK, int constrained,
                    const double* u, long long su, double* v, long long sv, void* stream) {
  SPK_RANGE("spk_stage_apply");
  if (int rc = check_level(c, level)) return rc;
  if (Q < 1 || Q > SPK_QMAX)
    return fail(SPK_EUNSUPPORTED, "fused stage operator supports Q in [1, 4], got " + std::to_string(Q));
  SpkApplyArgs a = base_args(c, level);
  a.u = u; a.v = v; a.su = su; a.sv = sv;
  a.constrained = constrained;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j < Q; ++j) {
      a.DM[i][j] = DM[i * Q + j];
      a.DK[i][j] = DK[i * Q + j];
    }
  return launch_apply(c, Q, false, EPI_STORE, a, (cudaStream_t)stream);
}

int spk_stage_apply_slab(spk_ctx* c, int level, int Q, const double* DM, const double* DK,
                         const double* u, long long su, double* v, long long sv, int x_elems,
                         int ex_begin, int ex_end, int store_last, void* stream) {
  SPK_RANGE("spk_stage_apply_slab");
  if (int rc = check_level(c, level)) return rc;
  if (c->dim != 3) return fail(SPK_ECONFIG, "slab windows need a 3D hierarchy");
  if (Q < 1 || Q > SPK_QMAX)
    return fail(SPK_EUNSUPPORTED, "fused stage operator supports Q in [1, 4], got " + std::to_string(Q));
  if (x_elems < 1 || ex_begin < 0 || ex_end > x_elems || ex_begin >= ex_end)
    return fail(SPK_ECONFIG, "bad slab element window");
  SpkApplyArgs a = base_args(c, level);
  a.g.Ex = x_elems;
  a.g.nx = c->K * x_elems + 1;
  a.g.n = (long long)a.g.nx * a.g.ny * a.g.nz;
  a.u = u; a.v = v; a.su = su; a.sv = sv;
  a.ex_begin = ex_begin; a.ex_end = ex_end; a.store_last = store_last;
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j < Q; ++j) {
      a.DM[i][j] = DM[i * Q + j];
      a.DK[i][j] = DK[i * Q + j];
    }
  return launch_apply(c, Q, false, EPI_STORE, a, (cudaStream_t)stream);
}

int spk_block_apply(spk_ctx* c, int level, int nblk, const double* lams, int lam_uniform, double tau,
                    int constrained, const double* u, long long su, double* v, long long sv,
                    void* stream) {
  SPK_RANGE("spk_block_apply");
  if (int rc = check_level(c, level)) return rc;
  if (nblk < 1) return SPK_OK;
  SpkApplyArgs a = base_args(c, level);
  a.u = u; a.v = v; a.su = su; a.sv = sv;
  return apply_blocks_chunked(c, level, nblk, lams, lam_uniform, tau, constrained, EPI_STORE, a,
                              (cudaStream_t)stream, nullptr, nullptr);
}

int spk_pair_apply(spk_ctx* c, int level, double re, double im, double tau, int constrained,
                   const double* u, double* v, void* stream) {
  SPK_RANGE("spk_pair_apply");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  SpkApplyArgs a = base_args(c, level);
  a.u = u; a.v = v; a.su = n; a.sv = n;
  a.constrained = constrained;
  a.DM[0][0] = re; a.DM[0][1] = -im; a.DM[1][0] = im; a.DM[1][1] = re;
  a.DK[0][0] = tau; a.DK[1][1] = tau;
  return launch_apply(c, 2, false, EPI_STORE, a, (cudaStream_t)stream);
}

int spk_residual(spk_ctx* c, int level, int nblk, const double* lams, double tau, const double* x,
                 const double* b, double* r, double* d_out, const double* c2s, void* stream) {
  SPK_RANGE("spk_residual");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  SpkApplyArgs a = base_args(c, level);
  a.u = x; a.su = n; a.b = b; a.r = r; a.d_out = d_out; a.se = n;
  return apply_blocks_chunked(c, level, nblk, lams, 0, tau, 1, EPI_RESID, a, (cudaStream_t)stream,
                              nullptr, d_out ? c2s : nullptr);
}

int spk_cheb_init(spk_ctx* c, int level, int nblk, const double* lams, double tau, const double* cs,
                  const double* b, double* r, double* x, double* d, void* stream) {
  SPK_RANGE("spk_cheb_init");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  for (int b0 = 0; b0 < nblk; b0 += SPK_BMAX) {
    const int nb = std::min(SPK_BMAX, nblk - b0);
    SpkRowArgs a = row_args(c, level);
    a.nblk = nb;
    a.tau = tau;
    for (int i = 0; i < nb; ++i) { a.lam[i] = lams[b0 + i]; a.c1[i] = cs[b0 + i]; }
    const long long off = (long long)b0 * n;
    a.b = b + off; a.r = r + off; a.x = x + off; a.d_out = d + off;
    cudaError_t e = spk_launch_cheb_rows(c->K, 0, a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cheb_init");
  }
  return SPK_OK;
}

int spk_cheb_start(spk_ctx* c, int level, int nblk, const double* lams, double tau, const double* thetas,
                   const double* b, double* d, void* stream) {
  SPK_RANGE("spk_cheb_start");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  for (int b0 = 0; b0 < nblk; b0 += SPK_BMAX) {
    const int nb = std::min(SPK_BMAX, nblk - b0);
    SpkRowArgs a = row_args(c, level);
    a.nblk = nb;
    a.tau = tau;
    for (int i = 0; i < nb; ++i) { a.lam[i] = lams[b0 + i]; a.c1[i] = thetas[b0 + i]; }
    const long long off = (long long)b0 * n;
    a.b = b + off; a.d_out = d + off;
    cudaError_t e = spk_launch_cheb_rows(c->K, 3, a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cheb_start");
  }
  return SPK_OK;
}

int spk_cheb_first_step(spk_ctx* c, int level, int nblk, const double* lams, double tau, const double* c1s,
                        const double* c2s, const double* b, const double* d_in, double* r, double* x,
                        double* d_out, int final_step, int* nan_flag, void* stream) {
  SPK_RANGE("spk_cheb_first_step");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  SpkApplyArgs ap = base_args(c, level);
  ap.u = d_in; ap.su = n; ap.v = d_out; ap.sv = n;
  if (int rc = apply_blocks_chunked(c, level, nblk, lams, 0, tau, 1, EPI_STORE, ap, (cudaStream_t)stream,
                                    nullptr, nullptr))
    return rc;
  for (int b0 = 0; b0 < nblk; b0 += SPK_BMAX) {
    const int nb = std::min(SPK_BMAX, nblk - b0);
    SpkRowArgs a = row_args(c, level);
    a.nblk = nb;
    a.tau = tau;
    a.final_step = final_step;
    a.nan_flag = nan_flag;
    for (int i = 0; i < nb; ++i) {
      a.lam[i] = lams[b0 + i];
      a.c1[i] = c1s[b0 + i];
      a.c2[i] = c2s[b0 + i];
    }
    const long long off = (long long)b0 * n;
    a.w = d_out + off; a.d = d_in + off; a.b = b + off; a.r = r + off; a.x = x + off; a.d_out = d_out + off;
    cudaError_t e = spk_launch_cheb_rows(c->K, final_step ? 5 : 4, a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cheb first update");
  }
  return SPK_OK;
}

int spk_cheb_split(spk_ctx* c, int level, int nblk) {
  if (int rc = check_level(c, level)) return -rc;
  return cheb_split(c, level, nblk) ? 1 : 0;
}

int spk_cheb_step(spk_ctx* c, int level, int nblk, const double* lams, double tau, const double* c1s,
                  const double* c2s, const double* d_in, double* r, double* x, double* d_out,
                  int final_step, int* nan_flag, void* stream) {
  SPK_RANGE("spk_cheb_step");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  if (cheb_split(c, level, nblk)) {
    // w = A d into d_out (constrained: boundary rows carry d), then the pointwise update
    SpkApplyArgs ap = base_args(c, level);
    ap.u = d_in; ap.su = n; ap.v = d_out; ap.sv = n;
    if (int rc = apply_blocks_chunked(c, level, nblk, lams, 0, tau, 1, EPI_STORE, ap, (cudaStream_t)stream,
                                      nullptr, nullptr))
      return rc;
    for (int b0 = 0; b0 < nblk; b0 += SPK_BMAX) {
      const int nb = std::min(SPK_BMAX, nblk - b0);
      SpkRowArgs a = row_args(c, level);
      a.nblk = nb;
      a.tau = tau;
      a.final_step = final_step;
      a.nan_flag = nan_flag;
      for (int i = 0; i < nb; ++i) {
        a.lam[i] = lams[b0 + i];
        a.c1[i] = c1s[b0 + i];
        a.c2[i] = c2s[b0 + i];
      }
      const long long off = (long long)b0 * n;
      a.w = d_out + off; a.d = d_in + off; a.r = r + off; a.x = x + off; a.d_out = d_out + off;
      cudaError_t e = spk_launch_cheb_rows(c->K, final_step ? 2 : 1, a, (cudaStream_t)stream);
      if (e != cudaSuccess) return cuda_fail(e, "cheb update");
    }
    return SPK_OK;
  }
  SpkApplyArgs a = base_args(c, level);
  a.u = d_in; a.su = n; a.r = r; a.x = x; a.d_out = d_out; a.se = n;
  a.final_step = final_step; a.nan_flag = nan_flag;
  return apply_blocks_chunked(c, level, nblk, lams, 0, tau, 1, EPI_CHEB, a, (cudaStream_t)stream, c1s,
                              c2s);
}

int spk_pair_residual(spk_ctx* c, int level, double re, double im, double tau, const double* x,
                      const double* b, double* r, double* d_out, double c2, void* stream) {
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  SpkApplyArgs a = base_args(c, level);
  a.u = x; a.su = n; a.b = b; a.r = r; a.d_out = d_out; a.se = n;
  a.constrained = 1;
  a.DM[0][0] = re; a.DM[0][1] = -im; a.DM[1][0] = im; a.DM[1][1] = re;
  a.DK[0][0] = tau; a.DK[1][1] = tau;
  a.tau = tau; a.jre = re; a.jim = im; a.c2[0] = c2;
  return launch_apply(c, 2, false, EPI_RESID, a, (cudaStream_t)stream);
}

int spk_pair_cheb_init(spk_ctx* c, int level, double re, double im, double tau, double cc,
                       const double* b, double* r, double* x, double* d, void* stream) {
  if (int rc = check_level(c, level)) return rc;
  SpkVecArgs a;
  std::memset(&a, 0, sizeof(a));
  a.g = c->dims[level];
  a.t = c->tabs[level];
  a.nblk = 2; a.constrained = 1; a.pair = 1;
  a.tau = tau; a.jre = re; a.jim = im; a.c[0] = cc;
  a.in0 = b; a.out0 = r; a.out1 = x; a.out2 = d;
  cudaError_t e = spk_launch_cheb_init(c->K, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "pair cheb_init");
  return SPK_OK;
}

int spk_pair_cheb_step(spk_ctx* c, int level, double re, double im, double tau, double c1, double c2,
                       const double* d_in, double* r, double* x, double* d_out, int final_step,
                       int* nan_flag, void* stream) {
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  SpkApplyArgs a = base_args(c, level);
  a.u = d_in; a.su = n; a.r = r; a.x = x; a.d_out = d_out; a.se = n;
  a.final_step = final_step; a.nan_flag = nan_flag;
  a.constrained = 1;
  a.DM[0][0] = re; a.DM[0][1] = -im; a.DM[1][0] = im; a.DM[1][1] = re;
  a.DK[0][0] = tau; a.DK[1][1] = tau;
  a.tau = tau; a.jre = re; a.jim = im; a.c1[0] = c1; a.c2[0] = c2;
  return launch_apply(c, 2, false, EPI_CHEB, a, (cudaStream_t)stream);
}

int spk_dinv_norm(spk_ctx* c, int level, int pair, double lam_or_re, double im, double tau,
                  const double* u, double* w, double* norm_dev, void* stream) {
  SPK_RANGE("spk_dinv_norm");
  if (int rc = check_level(c, level)) return rc;
  const long long n = c->dims[level].n;
  SpkApplyArgs a = base_args(c, level);
  a.u = u; a.v = w; a.su = n; a.sv = n;
  a.constrained = 1;
  a.tau = tau;
  int nctas = 0;
  // size the partial buffer conservatively before launching
  if (int rc = ensure_scratch(c, 1 << 16)) return rc;
  a.partial = c->partial;
  int rc;
  if (!pair) {
    a.nblk = 1; a.blk_base = 0; a.lam_uniform = 1; a.lam[0] = lam_or_re;
      rc = launch_apply(c, 1, true, EPI_DINV, a, (cudaStream_t)stream, &nctas);
  } else {
    a.DM[0][0] = lam_or_re; a.DM[0][1] = -im; a.DM[1][0] = im; a.DM[1][1] = lam_or_re;
    a.DK[0][0] = tau; a.DK[1][1] = tau;
    a.jre = lam_or_re; a.jim = im;
      rc = launch_apply(c, 2, false, EPI_DINV, a, (cudaStream_t)stream, &nctas);
  }
  if (rc) return rc;
  if (nctas > c->partial_cap) return fail(SPK_ECUDA, "partial buffer too small");
  cudaError_t e = spk_launch_reduce_partials(c->partial, nctas, norm_dev, 1, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "reduce_partials");
  return SPK_OK;
}

int spk_transfer(spk_ctx* c, int level, int nblk, int prolong, const double* in, double* out,
                 double* scratch, int accumulate, int mask, void* stream) {
  SPK_RANGE("spk_transfer");
  if (int rc = check_level(c, level)) return rc;
  if (level < 1) return fail(SPK_ECONFIG, "transfer needs level >= 1");
  const SpkDims gf = c->dims[level], gc = c->dims[level - 1];
  const int nf = gf.nz, nc = gc.nz, Nc = gc.Ez;
  const int dim = c->dim;
  // sweep order z (last axis), y, x; arrays are [nblk][x][y][z]; along x the levels may be slab
  // windows (local planes, global offsets x0; only the owned output planes are produced)
  int sx = prolong ? (dim >= 3 ? gc.nx : 1) : (dim >= 3 ? gf.nx : 1);
  int sy = prolong ? (dim >= 2 ? nc : 1) : (dim >= 2 ? nf : 1);
  int sz = prolong ? nc : nf;
  const int tz = prolong ? nf : nc;
  // scratch holds two ping-pong intermediates of at most nblk * max(local fine, local coarse) DoFs
  const long long half = (long long)nblk * (gf.n > gc.n ? gf.n : gc.n);
  double* bufA = scratch;
  double* bufB = scratch + half;
  const double* src = in;
  SpkTransferArgs a;
  std::memset(&a, 0, sizeof(a));
  a.prolong = prolong;
  for (int f = 0; f <= 2 * c->K; ++f)
    for (int j = 0; j <= c->K; ++j) a.P[f * (SPK_KMAX + 1) + j] = c->P[f * (SPK_KMAX + 1) + j];
  const SpkDims gout = prolong ? gf : gc;
  const int lout = prolong ? level : level - 1;
  // whole-mesh cubic 3D levels: one fused launch (vecops.cu prolong3d_kernel / restrict3d_kernel)
  // (restriction only on launch-bound levels: on large ones its fine-tile halo re-reads make the
  // three streaming sweeps faster, measured: C4 finest level 399 vs 950 us)
  const bool fuse_r = (long long)nblk * gf.n <= c->fuse_restrict_max;
  if (dim == 3 && c->fuse_transfer && (prolong || fuse_r) && whole_level(c, level) && whole_level(c, level - 1) &&
      gc.Ex == gc.Ey && gc.Ex == gc.Ez) {
    a.in = in; a.out = out; a.accumulate = accumulate; a.mask = mask; a.g = gout; a.Nc = Nc;
    cudaError_t e = prolong ? spk_launch_prolong3d(c->K, nblk, a, (cudaStream_t)stream)
                            : spk_launch_restrict3d(c->K, nblk, a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "fused transfer");
    return SPK_OK;
  }
  int nsweeps = dim;
  for (int sw = 0; sw < nsweeps; ++sw) {
    const bool last = (sw == nsweeps - 1);
    double* dst = last ? out : (sw % 2 == 0 ? bufA : bufB);
    a.in = src;
    a.out = dst;
    a.accumulate = last ? accumulate : 0;
    a.mask = last ? mask : 0;
    a.g = gout;
    a.Nc = Nc;
    a.in_off = 0; a.out_off = 0; a.o_begin = 0;
    if (sw == 0) {  // z axis
      a.outer = (long long)nblk * sx * sy; a.inner = 1; a.nin = sz; a.nout = tz; a.onodes = tz;
      sz = tz;
    } else if (sw == 1) {  // y axis
      const int ty = prolong ? nf : nc;
      a.outer = (long long)nblk * sx; a.inner = sz; a.nin = sy; a.nout = ty; a.onodes = ty;
      sy = ty;
    } else {  // x axis: windowed
      const SpkDims gi = prolong ? gc : gf;
      a.Nc = gc.Exg;
      a.outer = nblk; a.inner = (long long)sy * sz; a.nin = sx;
      a.in_off = gi.x0; a.out_off = gout.x0;
      a.onodes = gout.nx;
      a.o_begin = c->K * c->ex_begin[lout];
      a.nout = c->K * (c->ex_end[lout] - c->ex_begin[lout]) +
               ((c->store_last[lout] && c->ex_end[lout] == gout.Ex) ? 1 : 0);
      sx = gout.nx;
    }
    cudaError_t e = spk_launch_transfer(c->K, a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "transfer");
    src = dst;
  }
  return SPK_OK;
}

int spk_axpy_flag(long long total, double* x, const double* d, int* flag, void* stream) {
  cudaError_t e = spk_launch_axpy_flag(total, x, d, flag, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "axpy_flag");
  return SPK_OK;
}

int spk_combine(spk_ctx* c, int mask_level, long long n, int nin, int nout, const double* D,
                const double* in, long long sin, double* out, long long sout, int accumulate,
                void* stream) {
  SPK_RANGE("spk_combine");
  if (nin < 1 || nout < 1 || nin > SPK_CMAX || nout > SPK_CMAX)
    return fail(SPK_EUNSUPPORTED, "combine supports up to 18 rows/columns");
  SpkCombineArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int j = 0; j < nin; ++j) a.in[j] = in + j * sin;
  a.out = out; a.n = n; a.sin = sin; a.sout = sout;
  a.nin = nin; a.nout = nout; a.accumulate = accumulate;
  if (mask_level >= 0) {
    if (int rc = check_level(c, mask_level)) return rc;
    a.mask = 1;
    a.g = c->dims[mask_level];
  }
  for (int o = 0; o < nout; ++o)
    for (int j = 0; j < nin; ++j) a.D[o * SPK_CMAX + j] = D[o * nin + j];
  cudaError_t e = spk_launch_combine(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "combine");
  return SPK_OK;
}

int spk_peer_combine(long long n, int nin, const double* const* in_rows, int nout, const double* D,
                     double* out, long long sout, int accumulate, void* stream) {
  SPK_RANGE("spk_peer_combine");
  if (nin < 1 || nout < 1 || nin > SPK_CMAX || nout > SPK_CMAX)
    return fail(SPK_EUNSUPPORTED, "peer combine supports up to 18 rows/columns");
  SpkCombineArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int j = 0; j < nin; ++j) a.in[j] = in_rows[j];
  a.out = out; a.n = n; a.sout = sout;
  a.nin = nin; a.nout = nout; a.accumulate = accumulate;
  for (int o = 0; o < nout; ++o)
    for (int j = 0; j < nin; ++j) a.D[o * SPK_CMAX + j] = D[o * nin + j];
  cudaError_t e = spk_launch_combine(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "peer combine");
  return SPK_OK;
}

int spk_ipc_alloc(long long bytes, void** dev_ptr, void* handle) {
  if (!dev_ptr || !handle || bytes <= 0) return fail(SPK_ECONFIG, "bad ipc allocation request");
  cudaError_t e = cudaMalloc(dev_ptr, (size_t)bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(ipc window)");
  e = cudaMemset(*dev_ptr, 0, (size_t)bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(ipc window)");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, sizeof(h));
  return SPK_OK;
}

int spk_ipc_open(const void* handle, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return SPK_OK;
}

int spk_ipc_close(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return SPK_OK;
}

int spk_ipc_free(void* dev_ptr) {
  cudaError_t e = cudaFree(dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFree(ipc window)");
  return SPK_OK;
}

int spk_copy_d2d(void* dst, const void* src, long long bytes, void* stream) {
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
  return SPK_OK;
}

int spk_mgs(spk_ctx* c, long long n, double* w, const double* v_prev, const double* h_prev,
            const double* v_cur, double* out, void* stream) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  if (int rc = ensure_scratch(c, spk_mgs_grid())) return rc;
  SpkMgsArgs a;
  a.n = n; a.w = w; a.v_prev = v_prev; a.h_prev = h_prev; a.v_cur = v_cur; a.out = out;
  a.partial = c->partial; a.counter = c->counter; a.sq = 0;
  cudaError_t e = spk_launch_mgs(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mgs");
  return SPK_OK;
}

int spk_mgs_partial(spk_ctx* c, long long n, double* w, const double* v_prev, const double* h_prev,
                    const double* v_cur, double* out, void* stream) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  if (int rc = ensure_scratch(c, spk_mgs_grid())) return rc;
  SpkMgsArgs a;
  a.n = n; a.w = w; a.v_prev = v_prev; a.h_prev = h_prev; a.v_cur = v_cur; a.out = out;
  a.partial = c->partial; a.counter = c->counter; a.sq = 1;
  cudaError_t e = spk_launch_mgs(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mgs_partial");
  return SPK_OK;
}

int spk_band_axis(long long A, int nin, int nout, long long B, const int* col0, const double* vals, int bw,
                  const double* in, double* out, int accumulate, void* stream) {
  if (A < 1 || B < 1 || nin < 1 || nout < 1 || bw < 1 || bw > nin) return fail(SPK_EDIM, "band_axis: bad shape");
  cudaError_t e = spk_launch_band_axis(A, nin, nout, B, col0, vals, bw, in, out, accumulate, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "band_axis");
  return SPK_OK;
}

int spk_gauss_l2(spk_ctx* c, int dim, int ng, const double* ug, const double* w1, const double* ue,
                 const double* s1, double T, double* out, void* stream) {
  if (!c) return fail(SPK_ECONFIG, "null context");
  if (dim < 1 || dim > 3 || ng < 1) return fail(SPK_EDIM, "gauss_l2: bad shape");
  if (!ue && !s1) return fail(SPK_ECONFIG, "gauss_l2: need u_exact values or a separable factor");
  if (int rc = ensure_scratch(c, spk_gauss_l2_grid())) return rc;
  cudaError_t e = spk_launch_gauss_l2(dim, ng, ug, w1, ue, s1, T, c->partial, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "gauss_l2");
  return SPK_OK;
}

int spk_givens(const double* hcol, double* rcol, double* cs, double* g, double* res, int j, void* stream) {
  if (j < 0) return fail(SPK_ECONFIG, "givens: bad column");
  cudaError_t e = spk_launch_givens(hcol, rcol, cs, g, res, j, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "givens");
  return SPK_OK;
}

int spk_fp64_probe(int ctas, int threads, int iters, double* sink, void* stream) {
  if (ctas < 1 || threads < 32 || threads > 1024 || iters < 1) return fail(SPK_ECONFIG, "fp64_probe: bad sizes");
  cudaError_t e = spk_launch_fp64_probe(ctas, threads, iters, sink, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fp64_probe");
  return SPK_OK;
}

int spk_sqrt_dev(double* x, int count, void* stream) {
  if (count < 0 || count > 32) return fail(SPK_ECONFIG, "sqrt_dev: count must lie in [0, 32]");
  cudaError_t e = spk_launch_sqrt(x, count, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sqrt");
  return SPK_OK;
}

int spk_coarse_vcycle_level(spk_ctx* c) {
  if (!c || c->dim < 2) return -1;
  int best = -1;
  for (int l = 1; l <= c->max_level && l <= SPK_CV_LMAX; ++l) {
    if (!whole_level(c, l) || !whole_level(c, l - 1)) break;
    if (spk_coarse_vcycle_smem(c->K, l, c->dim) > SPK_CV_SMEM_MAX || c->dims[l].n > c->cv_max_nodes) break;
    best = l;
  }
  return best;
}

int spk_coarse_vcycle(spk_ctx* c, int lc, int nblk, const double* lams, double tau, int deg, const double* coef,
                      const double* cinv, const double* b, double* x, double* scratch, int* flags, void* stream) {
  SPK_RANGE("spk_coarse_vcycle");
  if (!c) return fail(SPK_ECONFIG, "null context");
  if (lc < 1 || lc > spk_coarse_vcycle_level(c)) return fail(SPK_ECONFIG, "coarse_vcycle: level not fusable");
  if (nblk < 1 || nblk > SPK_BMAX || deg < 1 || deg > 8) return fail(SPK_ECONFIG, "coarse_vcycle: bad sizes");
  SpkCoarseArgs a;
  std::memset(&a, 0, sizeof(a));
  a.lc = lc; a.nblk = nblk; a.deg = deg; a.tau = tau; a.dim = c->dim;
  a.top_in_smem = (spk_coarse_vcycle_smem(c->K, lc, c->dim) + spk_coarse_vcycle_top_bytes(c->K, lc, c->dim) <=
                   SPK_CV_SMEM_MAX && std::getenv("SPK_CV_TOP_GLOBAL") == nullptr) ? 1 : 0;
  for (int i = 0; i < nblk; ++i) a.lam[i] = lams[i];
  for (int l = 0; l <= lc; ++l) {  // M = h^d M_hat, K = h^(d-2) K_hat on the reference tables
    a.hd[l] = std::pow(c->h[l], c->dim);
    a.hk[l] = std::pow(c->h[l], c->dim - 2);
  }
  for (int f = 0; f <= 2 * c->K; ++f)
    for (int j = 0; j <= c->K; ++j) a.P[f * (SPK_KMAX + 1) + j] = c->P[f * (SPK_KMAX + 1) + j];
  if (!scratch) return fail(SPK_ECONFIG, "coarse_vcycle: scratch (nblk * 3 * n_lc doubles) required");
  a.coef = coef; a.cinv = cinv; a.b = b; a.x = x; a.flags = flags; a.scratch = scratch;
  a.sb = c->dims[lc].n; a.sx = c->dims[lc].n;
  cudaError_t e = spk_launch_coarse_vcycle(c->K, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "coarse_vcycle");
  return SPK_OK;
}

int spk_mgs_column(spk_ctx* c, long long n, int j, const double* const* basis, double* w, double* hcol,
                   double* v_next, void* stream) {
  SPK_RANGE("spk_mgs_column");
  // column j of modified Gram-Schmidt (krylov.py:74-82) as one call: j+2 fused sweeps, then
  // v_{j+1} = w / h_{j+1,j}; hcol points at H[0, j] (H[i, j] = hcol[i], device-resident)
  if (!c) return fail(SPK_ECONFIG, "null context");
  if (j < 0 || !basis || !w || !hcol) return fail(SPK_ECONFIG, "mgs_column: bad arguments");
  // small vectors: the whole column in one cooperative launch (the j+2 launches are latency-bound)
  if (c->mgs_coop && n <= c->mgs_coop_max && j + 1 < SPK_MGS_MAXCOL) {
    if (int rc = ensure_scratch(c, 6 * spk_mgs_coop_grid())) return rc;
    SpkMgsColArgs a;
    std::memset(&a, 0, sizeof(a));
    a.n = n; a.j = j; a.w = w; a.hcol = hcol; a.v_next = v_next; a.partial = c->partial;
    a.pair = (c->mgs_pair & 2) ? 1 : 0;  // SPK_MGS_PAIR bit 1: paired sweeps in the cooperative column too
    for (int i = 0; i <= j; ++i) a.basis[i] = basis[i];
    cudaError_t e = spk_launch_mgs_column_coop(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "mgs_column_coop");
    return SPK_OK;
  }
  if ((c->mgs_pair & 1) && j >= 1) {
    // paired sweeps (vecops.cu mgs2_kernel): pairs (v0, v1), (v2, v3), ...; sweep p applies pair
    // p - 1's updates and takes pair p's dots; the last sweep applies the last pair and takes ||w||
    if (int rc = ensure_scratch(c, 3 * spk_mgs_grid())) return rc;
    const int nv = j + 1;
    for (int i0 = 0; i0 < nv + 2; i0 += 2) {  // i0: first vector of the current pair (>= nv: norm)
      SpkMgs2Args a;
      std::memset(&a, 0, sizeof(a));
      a.n = n; a.w = w; a.partial = c->partial; a.counter = c->counter;
      a.np = i0 == 0 ? 0 : std::min(2, nv - (i0 - 2));
      for (int k = 0; k < a.np; ++k) { a.vp[k] = basis[i0 - 2 + k]; a.hp[k] = hcol + i0 - 2 + k; }
      a.nc = i0 >= nv ? 0 : std::min(2, nv - i0);
      for (int k = 0; k < a.nc; ++k) { a.vc[k] = basis[i0 + k]; a.out[k] = hcol + i0 + k; }
      if (a.nc == 0) a.out[0] = hcol + nv;
      cudaError_t e = spk_launch_mgs2(a, (cudaStream_t)stream);
      if (e != cudaSuccess) return cuda_fail(e, "mgs2");
      if (a.nc == 0) break;
    }
    if (v_next) return spk_scale_div(n, w, hcol + j + 1, v_next, stream);
    return SPK_OK;
  }
  int rc = spk_mgs(c, n, w, nullptr, nullptr, basis[0], hcol, stream);
  for (int i = 1; rc == SPK_OK && i <= j; ++i) rc = spk_mgs(c, n, w, basis[i - 1], hcol + i - 1, basis[i], hcol + i, stream);
  if (rc == SPK_OK) rc = spk_mgs(c, n, w, basis[j], hcol + j, nullptr, hcol + j + 1, stream);
  if (rc == SPK_OK && v_next) rc = spk_scale_div(n, w, hcol + j + 1, v_next, stream);
  return rc;
}

int spk_scale_div(long long n, const double* w, const double* h, double* v, void* stream) {
  cudaError_t e = spk_launch_scale_div(n, w, h, v, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "scale_div");
  return SPK_OK;
}

int spk_lincomb(long long n, int k, const double* const* vs_dev, const double* y_dev, double* z,
                void* stream) {
  cudaError_t e = spk_launch_lincomb(n, k, vs_dev, y_dev, z, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "lincomb");
  return SPK_OK;
}

int spk_outer3(spk_ctx* c, int level, const double* g1_dev, double* out, void* stream) {
  if (int rc = check_level(c, level)) return rc;
  SpkSepArgs a;
  a.g = c->dims[level]; a.gx = g1_dev; a.out = out;
  cudaError_t e = spk_launch_outer3(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "outer3");
  return SPK_OK;
}

int spk_rhs(spk_ctx* c, int level, int Q, const double* g1_dev, const double* T, const double* Ainv,
            const double* ku, double* out, void* stream) {
  SPK_RANGE("spk_rhs");
  if (int rc = check_level(c, level)) return rc;
  if (Q < 1 || Q > SPK_CMAX) return fail(SPK_EUNSUPPORTED, "rhs: bad Q");
  SpkRhsArgs a;
  std::memset(&a, 0, sizeof(a));
  a.g = c->dims[level]; a.gx = g1_dev; a.ku = ku; a.out = out; a.Q = Q;
  for (int j = 0; j < Q; ++j) a.T[j] = T[j];
  for (int i = 0; i < Q; ++i)
    for (int j = 0; j < Q; ++j) a.Ainv[i * SPK_CMAX + j] = Ainv[i * Q + j];
  cudaError_t e = spk_launch_rhs(a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "rhs");
  return SPK_OK;
}

int spk_update(long long n, int Q, const double* k, const double* bw_dev, double tau, double* u,
               void* stream) {
  cudaError_t e = spk_launch_update(n, Q, k, bw_dev, tau, u, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "update");
  return SPK_OK;
}

int spk_mask(spk_ctx* c, int level, int nblk, double* u, double value, void* stream) {
  if (int rc = check_level(c, level)) return rc;
  const SpkDims g = c->dims[level];
  cudaError_t e = spk_launch_mask((long long)nblk * g.n, g, u, value, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mask");
  return SPK_OK;
}

}  // extern "C"
