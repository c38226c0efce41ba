/*
 * gridot_b200.h -- C ABI of the B200-native quantized-Wasserstein hot path.
 *
 * One shared library, paper_2506_00976_b200/csrc/libgridot_b200.so, exports
 * these entry points.  They replace the fine-resolution stages of the
 * reference Python package `gridot` (paths relative to the reference root
 * pkg/src/gridot/); INTEGRATION.md shows the ctypes binding the reference
 * would add to call them.
 *
 * Conventions
 *   - Plain C types only.  Device buffers are caller-owned (allocated by the
 *     caller, e.g. through PyTorch's caching allocator); `stream` is a
 *     cudaStream_t passed as void*.  Calls are stream-ordered and reentrant;
 *     there is no global mutable state.
 *   - Grids: `ndim` axes (1..GDT_MAX_DIM), fine lengths `dims[ndim]`, flat
 *     index axis-1-fastest (measures.py:3-6).  Kernels taking `kappa` require
 *     every dims[a] to be a multiple of kappa (callers pad first with
 *     gdt_pad_f64, the zero padding of measures.py:236-245).
 *   - Batched calls process `batch` independent pairs laid out
 *     [batch, cells] contiguously.
 *   - Return value: GDT_OK or a negative GDT_ERR_*; per-pair outcomes of the
 *     iterative stages are reported in an int32 status array (GDT_PAIR_*),
 *     mapped by the Python layer onto the reference exception classes
 *     (errors.py).  No C++ exception crosses the ABI.
 */
#ifndef GRIDOT_B200_H
#define GRIDOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GDT_MAX_DIM 4

enum {
    GDT_OK = 0,
    GDT_ERR_ARG = -1,          /* invalid argument (shape, kappa, p, ndim) */
    GDT_ERR_CUDA = -2,         /* CUDA launch / runtime error */
    GDT_ERR_NOMEM = -3,        /* host allocation failed */
    GDT_ERR_UNSUPPORTED = -4   /* valid request this build does not implement */
};

/* per-pair status codes of the iterative stages */
enum {
    GDT_PAIR_OK = 0,
    GDT_PAIR_ZERO_DENOM_ROW = 1,  /* ZeroDenominatorError, sinkhorn.py:125-128 */
    GDT_PAIR_ZERO_DENOM_COL = 2,  /* ZeroDenominatorError, sinkhorn.py:131-134 */
    GDT_PAIR_OVERFLOW = 3         /* NumericOverflowError, sinkhorn.py:88-98    */
};

/* simplex status codes (_simplex.py:26-28) */
enum { GDT_LP_OPTIMAL = 0, GDT_LP_PIVOT_LIMIT = 1, GDT_LP_DISCONNECTED = 2 };

/* precision / order modes */
enum {
    GDT_MODE_EXACT = 0,  /* fp64, reference summation order (bit-exact) */
    GDT_MODE_FAST = 1    /* fp32 mode of BASELINE.json: any order, fp32 where safe */
};

const char *gdt_version(void);
/* Human-readable text of the last error raised on the calling thread. */
const char *gdt_last_error(void);

/* ---- layout helpers -------------------------------------------------- */

/* Zero-pad every axis up to a multiple of kappa.  Replaces pad_measure,
 * measures.py:236-245.  out: [batch, prod(padded dims)]. */
int gdt_pad_f64(const double *in, double *out, int64_t batch, int ndim,
                const int64_t *dims, int kappa, void *stream);

/* ---- K1: SumPool ------------------------------------------------------ */

/* Block sums, accumulated in ascending fine flat index (bit-exact with
 * np.add.at).  Replaces coarsen_measure, measures.py:257-267.
 * fine: [batch, prod(dims)] -> coarse: [batch, prod(dims)/kappa^ndim]. */
int gdt_sumpool_f64(const double *fine, double *coarse, int64_t batch, int ndim,
                    const int64_t *dims, int kappa, void *stream);

/* gdt_sumpool_f64 plus per-block statistics of the same pass:
 * stats [batch, n, 3] = {smallest positive mass, largest positive mass,
 * number of positive cells} (+inf, -inf, 0 without support); stats may be
 * NULL.  The coarse-level primal stage reads them (scale-range checks,
 * b = 1 on the target support, the default xi). */
int gdt_sumpool_stats_f64(const double *fine, double *coarse, double *stats, int64_t batch,
                          int ndim, const int64_t *dims, int kappa, void *stream);

/* ---- K2: marginally weighted coarse cost C-bar ------------------------ */

/* C-bar_kl = sum_{x in X_k, y in Y_l} rho(x,y)^p mu_x nu_y / (mu~_k nu~_l);
 * entries with mu~_k nu~_l == 0 take centre_cost[k,l] and are flagged in
 * `unused`.  Replaces weighted_cost_matrix, costs.py:128-171.
 *   mu, nu        [batch, N]   fine masses (padded grid, N = prod(dims))
 *   mu_c, nu_c    [batch, n]   their SumPool (gdt_sumpool_f64)
 *   centre_cost   [n, n]       C-tilde (costs.py:121-125), shared by the batch
 *   cost_table    [max_sq+1]   rho^p of integer squared distance, required
 *                              when p is neither 1 nor 2 (NULL otherwise)
 *   out           [batch, n, n], unused [batch, n, n] (uint8; NULL skips the mask)
 * mode GDT_MODE_EXACT reproduces the reference's rounding order exactly;
 * GDT_MODE_FAST uses block moments for p == 2 (fp64) and fp32 FFMA tiles
 * otherwise. */
int gdt_weighted_cost(const double *mu, const double *nu, const double *mu_c,
                      const double *nu_c, const double *centre_cost,
                      const double *cost_table, int64_t max_sq, double *out,
                      uint8_t *unused, int64_t batch, int ndim, const int64_t *dims,
                      int kappa, double p, int mode, void *stream);

/* C-bar at pooling factor kappa_c = factor * kappa_f from the C-bar at
 * kappa_f (same padded grid): the numerator of costs.py:128-171 is additive
 * over the factor^d fine-level blocks of each coarse block,
 *   C-bar_KL = sum_{k in K, l in L} C-bar_kl mu~_k nu~_l / (mu~_K nu~_L),
 * so a second O(N^2) pass over the fine cells is not needed when both levels
 * are requested (fp64 arithmetic; the result carries the rounding of
 * cbar_fine, so the engine uses it in fp32 mode only).
 *   cbar_fine [batch, nf, nf], mu_cf, nu_cf [batch, nf]: level kappa_f
 *   mu_c, nu_c [batch, n], centre_cost [n, n], out [batch, n, n],
 *   unused [batch, n, n] (uint8, nullable): level kappa_c
 *   cdims_fine [ndim]: coarse grid of level kappa_f (multiples of factor) */
int gdt_weighted_cost_pool(const double *cbar_fine, const double *mu_cf, const double *nu_cf,
                           const double *mu_c, const double *nu_c, const double *centre_cost,
                           double *out, uint8_t *unused, int64_t batch, int ndim,
                           const int64_t *cdims_fine, int factor, void *stream);

/* ---- K5/K6: primal upscaling (IPF + pricing + TV) --------------------- */

/* Block-sparse primal upscaling of a coarse plan, refit by IPF to the fine
 * marginals, priced, plus the weighted-TV inner sums.  Replaces the body of
 * primal_upscaling_upper_bound, quantized.py:311-363, with ipf_fit,
 * sinkhorn.py:101-142, over the upscaled coupling of upscale_coupling,
 * quantized.py:119-159 -- the fine coupling is never materialised.
 *   mu, nu        [batch, N] fine masses (padded grid)
 *   mu_c, nu_c    [batch, n] their SumPool (gdt_sumpool_f64); nullable
 *   stats         [2, batch, n, 3] block statistics of mu then nu
 *                 (gdt_sumpool_stats_f64); nullable
 *   cbar          [batch, n, n] C-bar of the batch (gdt_weighted_cost); nullable.
 *                 With mu_c, nu_c, stats, cbar, tv_w and bmap, GDT_MODE_FAST
 *                 and a uniform kernel, the stage runs at the coarse level:
 *                 every scaling is a per-block quotient of the masses, so a
 *                 sweep is O(arcs); transport^p = the fitted coarse plan priced
 *                 by C-bar (whose numerator is sum mu_t nu_s C_ts); one fine
 *                 pass: the weighted TV
 *   tv_w          [N] tv_weights of the padded grid (measures.py:289-296); nullable
 *                 (the fine-level TV kernel reads it when given, else computes
 *                 the weights per cell with the same formula)
 *   bmap          [N] int32 coarse block of each padded cell (block_index_map,
 *                 measures.py:248-254); nullable.  Without any of these the
 *                 fine-level kernels run.
 *   arc_off       [batch+1]  pair b owns arcs [arc_off[b], arc_off[b+1])
 *   row_ptr       [batch, n+1]  per pair CSR over coarse rows (offsets
 *                 relative to arc_off[b]); arcs sorted by (row, col)
 *   row_arc_col, row_arc_mass   [total arcs]
 *   col_ptr       [batch, n+1]  CSC over coarse columns; entries sorted by
 *                 (col, row); col_arc_row, col_arc_mass [total arcs]
 *   kernel_w      [m, m] paired kernel weights (m = kappa^ndim; row = source
 *                 offset, col = target offset, quantized.py:95-103)
 *   kernel_uniform  non-zero when all kernel_w entries are equal
 *   xi            per-pair stop threshold; xi < 0 selects the reference
 *                 default 1e-9 * (|supp mu| + |supp nu|) (quantized.py:319-320)
 *   max_iter      sweep cap (>= 1)
 *   cost_table    [max_sq+1] rho^p by integer squared distance for pricing
 *                 (required when p is neither 1 nor 2, else may be NULL)
 *                 GDT_MODE_EXACT with a uniform kernel spreads each pair over a
 *                 thread-block cluster of floor(SMs / batch) <= 8 CTAs when the
 *                 coarse grid has >= 128 blocks and kappa is 2, 4 or 8 (every
 *                 unit sum still runs in the reference's order: results do not
 *                 depend on the cluster size); the environment variable
 *                 GRIDOT_IPF_CLUSTER=<1..8> forces the size (1: one CTA per pair)
 *   mode          GDT_MODE_EXACT: IPF in the reference's order, fp64 pricing
 *                 costs; GDT_MODE_FAST: same IPF, p = 1 pricing costs from
 *                 fp32 sqrt (transport term within ~1e-7)
 *   out           [batch, 8]: {transport_p, tv_inner_mu, tv_inner_nu,
 *                 marginal_gap, iterations, converged, support_count, spare}
 *                 where transport_p = sum fitted*cost (before ^(1/p)) and
 *                 tv_inner_* = sum w_i |hat_i - marg_i| (before the root)
 *   status        [batch] GDT_PAIR_*
 *   scratch       device workspace of gdt_primal_scratch_bytes() bytes */
int64_t gdt_primal_scratch_bytes(int64_t batch, int ndim, const int64_t *dims,
                                 int kappa, int kernel_uniform);
int gdt_primal_upscale(const double *mu, const double *nu, const double *mu_c,
                       const double *nu_c, const double *stats, const double *cbar,
                       const double *tv_w, const int32_t *bmap, const int64_t *arc_off,
                       const int32_t *row_ptr, const int32_t *row_arc_col,
                       const double *row_arc_mass, const int32_t *col_ptr,
                       const int32_t *col_arc_row, const double *col_arc_mass,
                       const double *kernel_w, int kernel_uniform, const double *xi,
                       int64_t max_iter, double p, int64_t batch, int ndim,
                       const int64_t *dims, int kappa, const double *cost_table,
                       int64_t max_sq, int mode, double *out, int32_t *status, void *scratch,
                       void *stream);

/* Generic IPF on an explicit CSR kernel (rows = sources) with its CSC twin;
 * per-row sums in ascending column, per-column sums in ascending row (the
 * order of scipy's csr/csc matvec).  Replaces ipf_fit, sinkhorn.py:101-142,
 * for sparse/dense kernels and the one-ring fallback of quantized.py:335-344.
 *   out_a [nr], out_b [nc], out_kb [nr], out_kta [nc]
 *   info  [4]: {iterations, marginal_gap, converged, spare}; status [1]. */
int gdt_ipf_csr(const int64_t *indptr, const int32_t *indices, const double *data,
                const int64_t *t_indptr, const int32_t *t_indices, const double *t_data,
                const double *mu, const double *nu, int64_t nr, int64_t nc, double xi,
                int64_t max_iter, double *out_a, double *out_b, double *out_kb,
                double *out_kta, double *info, int32_t *status, void *stream);

/* Pricing of a fitted COO coupling on a grid: sum_e (a[row_e]*mass_e)*b[col_e]
 * * rho(x_row, x_col)^p.  Replaces quantized.py:346-355 for explicit
 * couplings.  row/col are fine flat ids of the padded grid; a, b, are the
 * full-grid scaling vectors.  out [1] = the sum before ^(1/p). */
int gdt_price_coo(const int64_t *row, const int64_t *col, const double *mass,
                  int64_t nnz, const double *a, const double *b, const double *cost_table,
                  int64_t max_sq, double p, int ndim, const int64_t *dims, double *out,
                  void *stream);

/* Weighted-TV inner sums sum_i w_i |x_i - y_i| (weighted_tv,
 * measures.py:298-315, before the 1/p root).  `weights` [N] may be NULL, in
 * which case w_i = rho(centre, x_i)^p of the grid (tv_weights,
 * measures.py:289-295) is generated on the fly.  x, y [batch, N]; out [batch]. */
int gdt_weighted_tv_inner(const double *x, const double *y, int64_t batch, int ndim,
                          const int64_t *dims, double p, const double *weights,
                          double *out, void *stream);

/* ---- K7-K10: dual upscaling ------------------------------------------ */

/* f_ext_k = min_{l in supp} (C~[k, dst[l]] - g[l]) (quantized.py:504-505).
 *   g [batch, n] (entries past supp_len[b] ignored), dst [batch, n] int32,
 *   supp_len [batch], centre_cost [n, n], f_ext [batch, n]. */
int gdt_coarse_ctransform(const double *g, const int32_t *dst, const int32_t *supp_len,
                          const double *centre_cost, int64_t n, int64_t batch,
                          double *f_ext, void *stream);

/* d-linear (method 0) or nearest (method 1) extension of a potential given on
 * a full coarse lattice to the fine grid `dims` (unpadded; clamped
 * extrapolation).  `axes` (device) holds the sorted lattice coordinates of
 * each axis back to back (cdims[0] values, then cdims[1], ...); for the bounds
 * these are the block centres kappa*b + (kappa+1)/2.  Replaces
 * interpolate_potential, quantized.py:388-447 (bit-exact, no FMA). */
int gdt_interpolate(const double *coarse, double *fine, int64_t batch, int ndim,
                    const int64_t *dims, const int64_t *cdims, const double *axes, int method,
                    void *stream);

/* Grid c-transform out_j = min_i rho(x_i, x_j)^p - v_i on one grid (the
 * source and target point sets of dual_upscaling_lower_bound coincide, so the
 * "target" and "source" directions of c_transform, quantized.py:450-484, are
 * the same operator).  dtype 0 = fp64, 1 = fp32 arithmetic and `out` type;
 * in_dtype is the type of `v` (fp64 input with fp32 arithmetic is allowed).
 * p == 2 uses per-axis separability (O(d N^{d+1})); other p run a tiled
 * brute-force min-plus with costs rho^p read from `cost_table` (indexed by
 * the integer squared distance; required for every p != 2).
 * If `mass` and `dot_out` are non-NULL, also writes dot_out[b] =
 * sum_j out_j * mass_j in fp64 (the dual value terms, quantized.py:512). */
int gdt_ctransform_grid(const void *v, void *out, int64_t batch, int ndim,
                        const int64_t *dims, double p, int dtype, int in_dtype,
                        const double *cost_table, int64_t max_sq, const double *mass,
                        double *dot_out, void *scratch, int64_t scratch_bytes, void *stream);
int64_t gdt_ctransform_scratch_bytes(int64_t batch, int ndim, const int64_t *dims,
                                     double p, int dtype);

/* c-transform between arbitrary point clouds (CostSpec, costs.py:56-99):
 * direction 0 ("target"): out_j = min_i C(xs_i, xt_j) - v_i over ns sources;
 * direction 1 ("source"): out_i = min_j C(xs_i, xt_j) - v_j.  fp64, costs
 * from the sequential squared distance then ^(p/2) (p=1 sqrt, p=2 as is). */
int gdt_ctransform_points(const double *xs, const double *xt, int64_t ns, int64_t nt,
                          int ndim, double p, const double *v, int direction, double *out,
                          void *stream);

/* sum_i a_i * b_i per row of [batch, n] (fp64 block reduction). */
int gdt_batched_dot(const double *a, const double *b, int64_t batch, int64_t n,
                    double *out, void *stream);

/* CUDA-core peak probes (the measured roofline denominators of bench.py):
 * `blocks` CTAs x 256 threads x 8 independent FMA chains x 16 unrolled steps
 * x `iters` loop trips of fma.rn.f32 (GDT_PROBE_FFMA), packed fma.rn.f32x2
 * (GDT_PROBE_FFMA2) or fma.rn.f64 (GDT_PROBE_DFMA); `sink` is a 4-byte device
 * buffer.  gdt_probe_flops gives the FLOP count of one such launch. */
#define GDT_PROBE_FFMA 0
#define GDT_PROBE_FFMA2 1
#define GDT_PROBE_DFMA 2
int gdt_probe_peak(int kind, int64_t blocks, int64_t iters, float *sink, void *stream);
int64_t gdt_probe_flops(int kind, int64_t blocks, int64_t iters);
/* = gdt_probe_peak(GDT_PROBE_FFMA, ...) */
int gdt_probe_fp32(int64_t blocks, int64_t iters, float *sink, void *stream);
/* Dependent-add latency of the FP64 pipe: one warp adds `adds` doubles from
 * shared memory into one accumulator, ((0 + p0) + p1) + ... -- the chain of
 * an exact-order IPF unit sum (sinkhorn.py:120-136) -- and reports the SM
 * cycles it took in cycles[0] (device buffer, 8 bytes).  The latency floor of
 * a sweep of the exact IPF is this figure x the longest unit. */
int gdt_probe_dadd_chain(int64_t adds, long long *cycles, void *stream);

/* ---- host coarse LP (stays on the host, _simplex.py) ------------------ */

/* Primal network simplex with the reference's pivot rules (northwest-corner
 * start, block pricing with Bland fallback, exact subtree relabel,
 * _simplex.py:31-361).  Host memory.  C row-major [ns, nt]; bi/bj/bf
 * [ns+nt-1]; u [ns]; v [nt].  block_size/max_pivots <= 0 select the
 * reference defaults.  Returns GDT_LP_* (>= 0) or GDT_ERR_*. */
int gdt_transport_simplex(const double *C, const double *sup, const double *dem,
                          int64_t ns, int64_t nt, int64_t block_size, int64_t max_pivots,
                          double tol, int64_t *bi, int64_t *bj, double *bf, double *u,
                          double *v, int64_t *pivots);

/* Batch of `count` problems on `threads` host threads (<= 0: all cores).
 * Every per-problem buffer is passed as a pointer value in a uint64 array.
 * Costs: C[q] != 0 is a dense row-major ns x nt matrix; C[q] == 0 selects a
 * translation-invariant cost on a full coarse grid (grid_ndim[q] axes,
 * extents grid_dims[q*GDT_MAX_DIM + a], ns = nt = cells) read from table[q]
 * over offset vectors x_j - x_i (extent 2*cd_a - 1 per axis, axis 0 fastest):
 * the C-tilde and C-min matrices of costs.py:121-125/174-192 without the
 * n^2 matrix.  warm_from[q] = -1 solves job q from the northwest corner with
 * the reference's pivot sequence; warm_from[q] = w (w < q, same shape) starts
 * from the optimal basis of job w instead (any optimal basis gives the same
 * optimal value; the quantization bounds warm-start the C-bar and C-min LPs
 * from the C-tilde basis on the same marginals); if job w did not reach an
 * optimum, job q is solved cold from the northwest corner instead.  Jobs
 * chained by warm_from run in order on one worker.  status[q] = GDT_LP_* or GDT_ERR_*. */
int gdt_transport_simplex_many(int64_t count, const uint64_t *C, const uint64_t *table,
                               const int32_t *grid_ndim, const int64_t *grid_dims,
                               const uint64_t *sup, const uint64_t *dem, const int64_t *ns,
                               const int64_t *nt, const int64_t *warm_from, double tol,
                               const uint64_t *bi, const uint64_t *bj, const uint64_t *bf,
                               const uint64_t *u, const uint64_t *v, int32_t *status,
                               int64_t *pivots, int threads);

/* gdt_transport_simplex_many with hand-off flags (both nullable): job q waits
 * until ready[q] != 0 (the caller sets it from another thread once the job's
 * cost data is in host memory) and done[q] is set to 1 when its outputs and
 * status are final, so finished jobs can be consumed while the batch runs. */
int gdt_transport_simplex_many_flags(int64_t count, const uint64_t *C, const uint64_t *table,
                                     const int32_t *grid_ndim, const int64_t *grid_dims,
                                     const uint64_t *sup, const uint64_t *dem, const int64_t *ns,
                                     const int64_t *nt, const int64_t *warm_from, double tol,
                                     const uint64_t *bi, const uint64_t *bj, const uint64_t *bf,
                                     const uint64_t *u, const uint64_t *v, int32_t *status,
                                     int64_t *pivots, int threads, const int32_t *ready,
                                     int32_t *done);

/* ---- entropic bounds (sinkhorn.py:150-299) ------------------------------ */

/* Device scratch for gdt_entropic_fit / gdt_entropic_plan: the dense
 * support-restricted kernel [ns][nt] fp64 plus sweep vectors and partials. */
int64_t gdt_entropic_scratch_bytes(int64_t ns, int64_t nt);

/* Alternating scaling on the Gibbs kernel K = exp(-C / eps) of the cost
 * C_ij = |xs_i - xt_j|^p (ipf_fit, sinkhorn.py:101-142), restarted in the log
 * domain (sinkhorn.py:150-178) when a denominator vanishes or a scaling vector
 * leaves [1e-100, 1e100] (_run_scaling, sinkhorn.py:181-195).  Replaces
 * _run_scaling for reg_lower_bound / reg_upper_bound.
 *   xs [ns, d], xt [nt, d]   support coordinates (row-major fp64, device)
 *   mu [ns], nu [nt]         positive support masses
 *   xi, max_iter             stop threshold on the L1 marginal gap, sweep cap
 *   f [ns], g [nt]           out: eps*log(a), eps*log(b) (or the log-domain
 *                            potentials)
 *   info [4]                 out: {iterations, marginal_gap, converged,
 *                            log_domain}
 *   status [1]               out: GDT_PAIR_OK, or GDT_PAIR_OVERFLOW when the
 *                            log-domain potentials are not finite
 * Synchronises `stream` every few sweeps to test for convergence. */
int gdt_entropic_fit(const double *xs, const double *xt, int64_t ns, int64_t nt, int d,
                     double p, double eps, const double *mu, const double *nu, double xi,
                     int64_t max_iter, double *f, double *g, double *info, int32_t *status,
                     void *scratch, void *stream);

/* Pricing of the fitted plan P_ij = exp((f_i + g_j - C_ij) / eps)
 * (sinkhorn.py:268-276): mu_hat [ns] = row sums, nu_hat [nt] = column sums,
 * transport [1] = sum_ij P_ij C_ij (before the 1/p root). */
int gdt_entropic_plan(const double *xs, const double *xt, int64_t ns, int64_t nt, int d,
                      double p, double eps, const double *f, const double *g, double *mu_hat,
                      double *nu_hat, double *transport, void *scratch, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* GRIDOT_B200_H */
