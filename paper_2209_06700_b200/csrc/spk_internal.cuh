// Internal declarations shared by the sm_100a kernels and the C-ABI host layer.
//
// Layout contract (reference fem.py:124, 213-218): a level's DoFs are a
// C-order (x slowest, z fastest) tensor of n_ax^dim nodes; stage/block vectors are stacked
// (nblk, n) with a stage stride. Degenerate axes (dim < 3) are represented as axes of one
// node and zero elements, so one 3D kernel family serves dim = 1, 2, 3.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define SPK_KMAX 4       // highest Q_k degree with a compiled kernel
#define SPK_QMAX 4       // highest stage count of the fused stage-coupled kernel
#define SPK_BMAX 16      // per-launch block-parameter slots (block mode)
#define SPK_ZTAIL_MAX 160  // K1 Z-phase tail items (Q * segments * (rows - 16)) with a host order
#define SPK_THREADS 256
#define SPK_SMALL_WORK_HOST (1LL << 23)  // = SPK_SMALL_WORK (stage_apply.cuh): direct small-level kernel

struct SpkDims {
  int nx, ny, nz;   // nodes per axis (1 for a degenerate axis)
  int Ex, Ey, Ez;   // elements per axis (0 for a degenerate axis)
  long long n;      // nx*ny*nz
  // x-slab windows (mesh partition along x): local plane 0 is global plane x0 (may be negative:
  // padding planes of the first slab); the global mesh has nxg planes / Exg elements along x.
  // A whole-mesh level has x0 = 0, nxg = nx, Exg = Ex.
  int x0, nxg, Exg;
};

// 1D element tables of one level, scaled by h (mass) and 1/h (stiffness), and the per-node
// diagonal pattern of the assembled 1D matrices.
struct SpkTab {
  double Me[SPK_KMAX + 1][SPK_KMAX + 1];
  double Ke[SPK_KMAX + 1][SPK_KMAX + 1];
};

enum SpkEpi {
  EPI_STORE = 0,   // v = Op(u)                      (boundary rows: identity if constrained)
  EPI_RESID = 1,   // r = b - Op(u); optionally d = c2 * Dinv r
  EPI_CHEB = 2,    // fused Chebyshev step on (r, x, d)
  EPI_DINV = 3,    // w = Dinv * Op(u)  + sum of squares (power iteration)
};

struct SpkApplyArgs {
  const double* u;        // operator input (stage/block q at u + q*su)
  double* v;              // output (EPI_STORE / EPI_DINV)
  long long su, sv;
  SpkDims g;
  int xe_chunk, nchunks;  // x-chunking of the sliding window
  int chunk_auto;         // host: the launcher may re-chunk with the kernel's real occupancy
  int ex_begin, ex_end;   // element range in x whose nodes are produced (slab windows)
  int store_last;         // also produce the last vertex plane when ex_end == Ex
  // virtual x-split (block mode): the CTA's Q "blocks" are Q consecutive x-ranges of ONE block,
  // vplanes planes apart (su = sv = se = vplanes * plane); 0 = off
  int vplanes;
  int constrained;
  int nblk;               // block mode: number of independent blocks
  int blk_base;           // block mode: index of the first block of this launch
  // coupled mode: v_i = sum_j DM_ij M u_j + DK_ij K u_j
  double DM[SPK_QMAX][SPK_QMAX];
  double DK[SPK_QMAX][SPK_QMAX];
  int dm_identity;        // coupled mode: DM is the identity (scaled by h^d) -> cheaper mix
  // block mode: v_b = lam_b M u_b + tau K u_b   (lam_uniform: lam[0] for every block)
  double lam[SPK_BMAX];
  int lam_uniform;
  double tau;
  SpkTab t;
  // epilogue operands
  const double* b;        // EPI_RESID: rhs
  double* r;              // EPI_RESID out / EPI_CHEB in-out residual
  double* x;              // EPI_CHEB in-out iterate
  double* d_out;          // EPI_CHEB new search direction; EPI_RESID optional d
  long long se;           // stage stride of epilogue operands
  double c1[SPK_BMAX], c2[SPK_BMAX];  // Chebyshev coefficients per block (pair: slot 0)
  // Jacobi diagonal: block mode diag = lam_b*dm + tau*dk ; pair mode uses (re, im, tau)
  double jre, jim;
  double* partial;        // EPI_DINV: per-CTA partial sums (deterministic reduction)
  double hd, hk;          // host only: h^dim and h^(dim-2) folded into the mix by the launcher
  int final_step;         // EPI_CHEB: last step -> write x + d_new only (fused x + d), NaN flag
  int* nan_flag;
  // K1 Z-phase: order of the items past the first 16 rows (host-computed, conflict-free STS.128)
  unsigned char ztail[SPK_ZTAIL_MAX];
};

// ---- programmatic dependent launch (PDL) ------------------------------------------------------
// The V-cycle's small-level kernels are each a few microseconds; launched with the PDL attribute a
// kernel is scheduled while its predecessor in the stream still runs, executes its prologue
// (shared-memory tables), and waits in spk_pdl_wait() -- before its first global-memory access --
// until the predecessor has completed and its writes are visible. spk_pdl_trigger() lets the next
// kernel be scheduled early. Without the attribute both are no-ops.
__device__ __forceinline__ void spk_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void spk_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool spk_pdl_enabled();     // SPK_PDL=0 disables (api.cu)
long long spk_pdl_max_ctas();  // launches up to this many CTAs use the attribute (SPK_PDL_MAX)

template <typename... KArgs, typename... Args>
inline cudaError_t spk_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (spk_pdl_enabled() && (long long)grid.x * grid.y * grid.z <= spk_pdl_max_ctas()) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// launchers (stage_apply.cu)
cudaError_t spk_launch_apply(int K, int Q, bool block_mode, int epi, const SpkApplyArgs& a,
                             cudaStream_t s, int* nctas_out);
