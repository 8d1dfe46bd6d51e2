// Argument blocks of the memory-bound kernels (vecops.cu).
#pragma once
#include "spk_internal.cuh"

#define SPK_CMAX 18   // max rows/cols of a stage-combine matrix (2*ceil(9/2) = 10 real rows)

struct SpkVecArgs {
  SpkDims g;
  SpkTab t;
  int nblk, blk_base, constrained, pair, lam_uniform;
  double lam[SPK_BMAX];
  double tau, jre, jim;
  double c[SPK_BMAX];
  const double* in0;
  double* out0;
  double* out1;
  double* out2;
};

// row-parallel pointwise smoother kernels (one CTA row group per (x, y) line of nz nodes, all blocks):
// Chebyshev start and the Chebyshev update that follows a K1 STORE of w = A d
struct SpkRowArgs {
  SpkDims g;
  SpkTab t;
  int nblk, constrained, final_step;
  int row0, nrows;        // rows (x*ny + y) [row0, row0 + nrows): the owned planes of a slab window
  int tpr;                // threads per row (power of two, <= blockDim)
  double lam[SPK_BMAX], c1[SPK_BMAX], c2[SPK_BMAX];
  double tau;
  const double* w;        // update: A d
  const double* d;        // update: previous direction
  const double* b;        // init: right-hand side
  double* r;
  double* x;
  double* d_out;
  int* nan_flag;
};

struct SpkTransferArgs {
  const double* in;
  double* out;
  long long outer, inner;
  int nin, nout;
  int Nc;         // coarse elements along the axis (global)
  int in_off, out_off;  // global node index of local node 0 of input / output along the axis
  int o_begin;    // first local output node produced (nout nodes from there)
  int onodes;     // local output nodes along the axis (extent of the output array)
  int prolong;    // 1: coarse -> fine, 0: restriction (transpose)
  int accumulate; // out += result
  int mask;       // zero boundary nodes of level g (final sweep)
  SpkDims g;
  double P[(2 * SPK_KMAX + 1) * (SPK_KMAX + 1)];
};

#define SPK_MGS_MAXCOL 240
struct SpkMgsColArgs {  // one MGS column (spk_mgs_column) in one cooperative launch
  long long n;
  int j;
  double* w;
  double* hcol;     // H[0 .. j+1, j]
  double* v_next;   // w / H[j+1, j] (optional)
  double* partial;  // 2 * grid doubles (paired: 6 * grid)
  int pair;         // paired sweeps (two basis vectors per grid barrier)
  const double* basis[SPK_MGS_MAXCOL];
};

struct SpkCombineArgs {
  const double* in[SPK_CMAX];  // input rows (local rows, or rows in peer GPUs' memory)
  double* out;
  long long n, sin, sout;
  int nin, nout, mask, accumulate;
  SpkDims g;
  double D[SPK_CMAX * SPK_CMAX];
};

struct SpkMgsArgs {
  long long n;
  double* w;
  const double* v_prev;
  const double* h_prev;
  const double* v_cur;
  double* out;
  double* partial;
  unsigned* counter;
  int sq;  // v_cur == null: 1 -> *out = sum w^2 (a rank's partial, all-reduced by the caller), 0 -> ||w||
};

// paired MGS sweep: w -= h0 v_prev0 + h1 v_prev1 (in that order), then the dots of w with up to two
// further basis vectors and their mutual dot (or ||w||)
struct SpkMgs2Args {
  long long n;
  double* w;
  const double* vp[2];
  const double* hp[2];
  const double* vc[2];
  int np, nc;
  double* out[2];
  double* partial;   // 3 x grid
  unsigned* counter;
};
cudaError_t spk_launch_mgs2(const SpkMgs2Args& a, cudaStream_t s);

struct SpkSepArgs {
  SpkDims g;
  const double* gx;
  double* out;
};

struct SpkRhsArgs {
  SpkDims g;
  const double* gx;     // 1D load vector of the separable spatial factor
  const double* ku;     // K u_n
  double* out;          // (Q, n)
  int Q;
  double T[SPK_CMAX];   // time factors T(t_n + c_j tau)
  double Ainv[SPK_CMAX * SPK_CMAX];
};

cudaError_t spk_launch_cheb_init(int K, const SpkVecArgs& a, cudaStream_t s);
cudaError_t spk_launch_axpy_flag(long long total, double* x, const double* d, int* flag, cudaStream_t s);
cudaError_t spk_launch_cheb_rows(int K, int op, const SpkRowArgs& a, cudaStream_t s);
// fused coarse-level V-cycle (coarse_vcycle.cu): levels 0..lc of a whole-mesh 3D hierarchy, one CTA
// per block, all level vectors in shared memory
#define SPK_CV_LMAX 4
#define SPK_CV_SMEM_MAX (200 * 1024)
struct SpkCoarseArgs {
  int lc, nblk, deg, dim;  // dim: 2 or 3 (2D: degenerate x axis)
  int top_in_smem;         // level lc's x, b, r, d, w in shared memory (else global / L2)
  double tau;
  double lam[SPK_BMAX];                            // block shifts (unscaled)
  double hd[SPK_CV_LMAX + 1], hk[SPK_CV_LMAX + 1];  // h^dim, h^(dim-2) per level
  double P[(2 * SPK_KMAX + 1) * (SPK_KMAX + 1)];   // 1D prolongation table
  const double* coef;  // [lc+1][nblk][1 + 2(deg-1)]: theta, (c1, c2) per inner step
  const double* cinv;  // (nblk, n0, n0) row-major inverse of the constrained coarse operator
  const double* b;     // rhs at level lc, block stride sb
  double* x;           // result at level lc, block stride sx
  int* flags;          // per-level NaN flags
  double* scratch;     // (nblk, 3, n_lc): r, d, w of every level (global, L2-resident)
  long long sb, sx;
};
long long spk_coarse_vcycle_smem(int K, int lc, int dim);
long long spk_coarse_vcycle_top_bytes(int K, int lc, int dim);
cudaError_t spk_launch_coarse_vcycle(int K, const SpkCoarseArgs& a, cudaStream_t s);

cudaError_t spk_launch_transfer(int K, const SpkTransferArgs& a, cudaStream_t s);
cudaError_t spk_launch_prolong3d(int K, int nblk, const SpkTransferArgs& a, cudaStream_t s);
cudaError_t spk_launch_restrict3d(int K, int nblk, const SpkTransferArgs& a, cudaStream_t s);
cudaError_t spk_launch_combine(const SpkCombineArgs& a, cudaStream_t s);
int spk_mgs_grid();
cudaError_t spk_launch_mgs(const SpkMgsArgs& a, cudaStream_t s);
int spk_mgs_coop_grid();
cudaError_t spk_launch_mgs_column_coop(const SpkMgsColArgs& a, cudaStream_t s);
cudaError_t spk_launch_sqrt(double* x, int count, cudaStream_t s);
cudaError_t spk_launch_givens(const double* hcol, double* rcol, double* cs, double* g, double* res, int j,
                              cudaStream_t s);
cudaError_t spk_launch_band_axis(long long A, int nin, int nout, long long B, const int* col0, const double* vals,
                                 int bw, const double* in, double* out, int acc, cudaStream_t s);
int spk_gauss_l2_grid();
cudaError_t spk_launch_gauss_l2(int dim, int ng, const double* ug, const double* w1, const double* ue,
                                const double* s1, double T, double* partial, double* out, cudaStream_t s);
cudaError_t spk_launch_fp64_probe(int ctas, int threads, int iters, double* sink, cudaStream_t s);
cudaError_t spk_launch_scale_div(long long n, const double* w, const double* h, double* v, cudaStream_t s);
cudaError_t spk_launch_reduce_partials(const double* partial, int m, double* out, int sqrt_out, cudaStream_t s);
cudaError_t spk_launch_lincomb(long long n, int k, const double* const* vs, const double* y, double* z,
                               cudaStream_t s);
cudaError_t spk_launch_outer3(const SpkSepArgs& a, cudaStream_t s);
cudaError_t spk_launch_rhs(const SpkRhsArgs& a, cudaStream_t s);
cudaError_t spk_launch_update(long long n, int Q, const double* k, const double* bw, double tau, double* u,
                              cudaStream_t s);
cudaError_t spk_launch_mask(long long total, const SpkDims& g, double* u, double value, cudaStream_t s);
int spk_apply_smem_bytes(int K, int Q);
int spk_apply_geo(int K, int Q, int what);  // 0 smem bytes, 1 threads, 2 TYE, 3 TZE
