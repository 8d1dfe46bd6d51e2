/* spk.h - C-ABI of the B200-native stage-parallel Radau IIA hot path (libspk, sm_100a).
 *
 * Every entry point takes plain pointers and sizes; device pointers are fp64 CUDA buffers in the
 * reference layout: a level's DoFs are C-order (x slowest) n_ax^dim nodes, stage/block vectors
 * are stacked (nblk, n) with an element stride. All calls are ordered on the caller's stream
 * (cudaStream_t passed as void*). Return value: SPK_OK or one of the error codes below; the text
 * of the last error of the calling thread is in spk_last_error().
 *
 * Which reference interface each entry point replaces (file:line under the reference package
 * pkg/src/spirk/):
 *   spk_ctx_create          GridHierarchy.__init__ / build_hierarchy      fem.py:75-102, :300
 *   spk_level_info          GridLevel.n_per_axis/n_dofs/h                 fem.py:44-69
 *   spk_nodes_1d            GridLevel.axis_coords                         fem.py:68-69
 *   spk_stage_apply         (D_M (x) M + D_K (x) K) u, K1 stage operator   fem.py:120-151 + SPEC irk:A
 *   spk_block_apply         apply_shifted / apply_constrained             fem.py:145-170
 *   spk_pair_apply          PairBlockSolver._apply                        multigrid.py:292-304
 *   spk_residual            _VCycleBase._cycle r = b - A x               multigrid.py:122
 *   spk_cheb_init/step      ChebyshevSmoother.apply                       multigrid.py:74-88
 *   spk_pair_residual/cheb  PairBlockSolver smoothing (2x2 block Jacobi)  multigrid.py:306-313
 *   spk_dinv_norm           estimate_lambda_max inner step                multigrid.py:45-62
 *   spk_transfer            prolong / restrict (+ mask, + accumulate)     fem.py:189-211, multigrid.py:171-177
 *   spk_combine             SPEC tensor_ops dense_combine (D (x) I) u
 *   spk_mgs / spk_scale_div / spk_lincomb  gmres MGS, basis, final update  krylov.py:69-93
 *   spk_givens                            gmres least-squares residual       krylov.py:84-87, :106-110
 *   spk_band_axis / spk_gauss_l2          load_vector / l2_error            fem.py:220-273
 *   spk_mgs_partial / spk_sqrt_dev        gmres MGS with all-reduced dots   krylov.py:74-82 (+ PAPER.md:426-443)
 *   spk_rhs / spk_outer3 / spk_update      SPEC irk_solver.assemble_rhs / step
 *   spk_mask                GridHierarchy.constrain                       fem.py:153-158
 *   spk_peer_combine        SPEC tensor_ops sharedmem_combine (D (x) I) u
 *   spk_ipc_*               peer windows of the shared-memory backend     SPEC.md:354 (runtime DESIGN)
 *   spk_ctx_set_slab        (no reference code: the paper's spatial partition inside a stage
 *                           group; SPEC RankGrid partitions b)
 */
#ifndef SPK_H_
#define SPK_H_

#ifdef __cplusplus
extern "C" {
#endif

#define SPK_OK 0
#define SPK_EDIM 1          /* DimensionMismatchError */
#define SPK_ECONFIG 2       /* ConfigurationError */
#define SPK_ENUMERIC 3      /* NumericalFailureError */
#define SPK_ESPECTRAL 4     /* SpectralFailureError */
#define SPK_ECUDA 5         /* CUDA runtime failure */
#define SPK_ECOMM 6         /* collective failure */
#define SPK_EUNSUPPORTED 7  /* degree / stage count without a compiled kernel */

typedef struct spk_ctx spk_ctx;

int spk_version(void);
const char* spk_last_error(void);

/* host-side discretisation data (no GPU needed) */
int spk_ctx_create(int dim, int max_level, int degree, spk_ctx** out);
int spk_ctx_destroy(spk_ctx* ctx);
/* Turn level `level` of a 3D context into an x-slab window of the global 2^level-element mesh:
 * the local arrays hold x_elems elements along x (K*x_elems+1 planes) whose plane 0 is global
 * plane x0_plane (negative on the first slab: padding planes); every entry point at this level then
 * produces only the nodes of local elements [ex_begin, ex_end) (+ the last vertex plane if
 * store_last), with boundary rows, Jacobi classes and sources taken at global x positions.
 * Halo planes are the caller's (exchanged before each operator application). */
int spk_ctx_set_slab(spk_ctx* ctx, int level, int x_elems, int x0_plane, int ex_begin, int ex_end,
                     int store_last);
int spk_level_info(const spk_ctx* ctx, int level, int* n_per_axis, long long* n_dofs, double* h,
                   int* n_elems);
int spk_level_tables(const spk_ctx* ctx, int level, double* Me, double* Ke);
int spk_nodes_1d(const spk_ctx* ctx, int level, double* out);
int spk_prolong_table(const spk_ctx* ctx, double* P);
int spk_apply_smem(int degree, int Q);
int spk_set_chunks(spk_ctx* ctx, int target_ctas);

/* K1: v_i = sum_j (DM_ij M + DK_ij K) u_j, Q stages, DM/DK row-major Q x Q host arrays */
int spk_stage_apply(spk_ctx* ctx, int level, int Q, const double* DM, const double* DK, int constrained,
                    const double* u, long long su, double* v, long long sv, void* stream);
/* K1 on an x-slab with halo planes: the local array has x_elems elements along x (K*x_elems+1
 * planes); only nodes of elements [ex_begin, ex_end) (+ the last plane if store_last) are written */
int spk_stage_apply_slab(spk_ctx* ctx, int level, int Q, const double* DM, const double* DK,
                         const double* u, long long su, double* v, long long sv, int x_elems,
                         int ex_begin, int ex_end, int store_last, void* stream);
/* v_b = lam_b M u_b + tau K u_b for b < nblk (lams: nblk host values, or 1 if lam_uniform) */
int spk_block_apply(spk_ctx* ctx, int level, int nblk, const double* lams, int lam_uniform, double tau,
                    int constrained, const double* u, long long su, double* v, long long sv,
                    void* stream);
/* pair operator [[K',-M'],[M',K']] on (2, n): K' = re M + tau K, M' = im M */
int spk_pair_apply(spk_ctx* ctx, int level, double re, double im, double tau, int constrained,
                   const double* u, double* v, void* stream);

/* smoother building blocks (block mode: per-block lam / Chebyshev coefficients) */
int spk_residual(spk_ctx* ctx, int level, int nblk, const double* lams, double tau, const double* x,
                 const double* b, double* r, double* d_out, const double* c2s, void* stream);
int spk_cheb_init(spk_ctx* ctx, int level, int nblk, const double* lams, double tau, const double* cs,
                  const double* b, double* r, double* x, double* d, void* stream);
/* final_step != 0: fused last step, writes only x <- x + d_in + d_new and raises *nan_flag on NaN/Inf */
int spk_cheb_step(spk_ctx* ctx, int level, int nblk, const double* lams, double tau, const double* c1s,
                  const double* c2s, const double* d_in, double* r, double* x, double* d_out,
                  int final_step, int* nan_flag, void* stream);
int spk_pair_residual(spk_ctx* ctx, int level, double re, double im, double tau, const double* x,
                      const double* b, double* r, double* d_out, double c2, void* stream);
int spk_pair_cheb_init(spk_ctx* ctx, int level, double re, double im, double tau, double c,
                       const double* b, double* r, double* x, double* d, void* stream);
int spk_pair_cheb_step(spk_ctx* ctx, int level, double re, double im, double tau, double c1, double c2,
                       const double* d_in, double* r, double* x, double* d_out, int final_step,
                       int* nan_flag, void* stream);
/* power iteration step: w = Dinv A u, *norm_dev = ||w||_2 (device scalar); pair != 0 uses (re, im) */
int spk_dinv_norm(spk_ctx* ctx, int level, int pair, double lam_or_re, double im, double tau,
                  const double* u, double* w, double* norm_dev, void* stream);

/* transfers: prolong (coarse level -> level) or restrict (level -> level-1) for nblk blocks */
int spk_transfer(spk_ctx* ctx, int level, int nblk, int prolong, const double* in, double* out,
                 double* scratch, int accumulate, int mask, void* stream);
int spk_axpy_flag(long long total, double* x, const double* d, int* flag, void* stream);

/* (D (x) I) u with D row-major nout x nin (host); mask_level >= 0 zeroes its boundary nodes */
int spk_combine(spk_ctx* ctx, int mask_level, long long n, int nin, int nout, const double* D,
                const double* in, long long sin, double* out, long long sout, int accumulate,
                void* stream);

/* out_o = sum_j D[o, j] in_rows[j] over n entries; in_rows is a HOST array of nin device pointers,
 * which may point into peer GPUs' memory (CUDA IPC windows): the stage exchange and the combine
 * arithmetic are one kernel reading over NVLink (the shared-memory combine backend) */
int spk_peer_combine(long long n, int nin, const double* const* in_rows, int nout, const double* D,
                     double* out, long long sout, int accumulate, void* stream);
/* peer windows: cudaMalloc'd buffer + its 64-byte IPC handle; open / close a peer's window */
int spk_ipc_alloc(long long bytes, void** dev_ptr, void* handle64);
int spk_ipc_open(const void* handle64, void** dev_ptr);
int spk_ipc_close(void* dev_ptr);
int spk_ipc_free(void* dev_ptr);
int spk_copy_d2d(void* dst, const void* src, long long bytes, void* stream);
/* Chebyshev from a zero start without materialising r = b, x = 0 (large levels, see spk_cheb_split):
 * spk_cheb_start: d = Dinv b / theta; spk_cheb_first_step: w = A d (into d_out), r = b - w, x = d,
 * d_out = c1 d + c2 Dinv r (final_step: x = d + d_new only, NaN flag) */
int spk_cheb_start(spk_ctx* ctx, int level, int nblk, const double* lams, double tau, const double* thetas,
                   const double* b, double* d, void* stream);
int spk_cheb_first_step(spk_ctx* ctx, int level, int nblk, const double* lams, double tau, const double* c1s,
                        const double* c2s, const double* b, const double* d_in, double* r, double* x,
                        double* d_out, int final_step, int* nan_flag, void* stream);
/* single-block K1 launches on whole-mesh 3D levels sweep 4 (or 2) x-ranges per CTA (default on) */
int spk_set_vsplit(spk_ctx* ctx, int on);
/* Chebyshev steps run split on levels with at least min_block_dofs (blocks x DoFs; default 2^18) and
 * always for >= 3 blocks (measured faster than the fused K1 epilogue there) */
int spk_set_cheb_split(spk_ctx* ctx, long long min_block_dofs);
/* 1 if the Chebyshev steps of this level run split (K1 STORE + pointwise update), 0 if fused */
int spk_cheb_split(spk_ctx* ctx, int level, int nblk);
/* GMRES: w -= (*h_prev) v_prev ; *out = <v_cur, w>  (v_cur == NULL: *out = ||w||) */
int spk_mgs(spk_ctx* ctx, long long n, double* w, const double* v_prev, const double* h_prev,
            const double* v_cur, double* out, void* stream);
int spk_scale_div(long long n, const double* w, const double* h, double* v, void* stream);
/* Fused V-cycle on levels 0..lc (multigrid.py:110-140 with the direct coarse solve, block family):
 * x_lc = V-cycle(b_lc) for nblk blocks in one launch (one CTA per block, level vectors in shared
 * memory). coef: device [lc+1][nblk][1 + 2(deg-1)] (theta, then c1, c2 per inner Chebyshev step);
 * cinv: device (nblk, n0, n0) inverse of the constrained coarse operator; scratch: device
 * nblk * 3 * n_lc doubles (r, d, w); flags: device int per level.
 * spk_coarse_vcycle_level returns the highest fusable level (-1: none). */
int spk_coarse_vcycle_level(spk_ctx* ctx);
int spk_coarse_vcycle(spk_ctx* ctx, int lc, int nblk, const double* lams, double tau, int deg,
                      const double* coef, const double* cinv, const double* b, double* x, double* scratch,
                      int* flags, void* stream);
/* distributed MGS (krylov.py:74-82 with all-reduced inner products): same sweep as spk_mgs, but
 * with v_cur == NULL *out is this rank's sum of squares (the caller all-reduces it, then
 * spk_sqrt_dev turns the sum into the norm H[j+1, j]) */
int spk_mgs_partial(spk_ctx* ctx, long long n, double* w, const double* v_prev, const double* h_prev,
                    const double* v_cur, double* out, void* stream);
int spk_sqrt_dev(double* x, int count, void* stream);
/* GMRES least-squares residual on the device (krylov.py:84-87): column j of H (hcol, j+2 entries,
 * not modified) rotated by the previous Givens rotations (cs: 2 per column) into rcol, a new rotation
 * for H[j+1, j], g (the rotated beta e_1) updated, *res = |g[j+1]| = the lstsq residual norm */
int spk_givens(const double* hcol, double* rcol, double* cs, double* g, double* res, int j, void* stream);
/* Gauss-point quadrature (load_vector / l2_error, fem.py:220-273): a banded matrix (device col0[nout],
 * vals[nout][bw]) applied along one axis of a (A, nin, B) array, out (+)= ; and the L2 norm
 * sqrt(sum_g w(g) (ug(g) - u_exact(g))^2) over the ng^dim tensor Gauss grid, u_exact from the device
 * array ue or, with ue == NULL, the separable T * prod_d s1[g_d]; *out is a device scalar */
int spk_band_axis(long long A, int nin, int nout, long long B, const int* col0, const double* vals, int bw,
                  const double* in, double* out, int accumulate, void* stream);
int spk_gauss_l2(spk_ctx* ctx, int dim, int ng, const double* ug, const double* w1, const double* ue,
                 const double* s1, double T, double* out, void* stream);
/* FP64 pipe probe (no reference counterpart; measurement only): ctas x threads threads each run
 * 8 independent DFMA chains of 16 * iters steps = 256 * iters flops per thread; sink: >= threads
 * doubles of device scratch (never written in practice). Timed by the caller with CUDA events. */
int spk_fp64_probe(int ctas, int threads, int iters, double* sink, void* stream);
/* One MGS column (krylov.py:74-82) in one call: the j+2 fused spk_mgs sweeps of w against basis[0..j]
 * (host array of device pointers), H[0..j+1, j] written to hcol (device), then v_next = w / H[j+1, j]
 * when v_next is not NULL. Same launches and order as the per-sweep calls. */
int spk_mgs_column(spk_ctx* ctx, long long n, int j, const double* const* basis, double* w, double* hcol,
                   double* v_next, void* stream);
int spk_lincomb(long long n, int k, const double* const* vs_dev, const double* y_dev, double* z,
                void* stream);

/* separable fields and the stage right-hand side */
int spk_outer3(spk_ctx* ctx, int level, const double* g1_dev, double* out, void* stream);
int spk_rhs(spk_ctx* ctx, int level, int Q, const double* g1_dev, const double* T, const double* Ainv,
            const double* ku, double* out, void* stream);
int spk_update(long long n, int Q, const double* k, const double* bw_dev, double tau, double* u,
               void* stream);
int spk_mask(spk_ctx* ctx, int level, int nblk, double* u, double value, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPK_H_ */
