// Entropic bounds (reference sinkhorn.py:150-299): alternating scaling on the
// dense Gibbs kernel K = exp(-C / eps) of a point-cloud cost, its log-domain
// restart, and the pricing of the fitted plan.
//
// Layout: the support-restricted kernel is materialised once per fit in the
// caller's scratch as fp64 [ns][nt] row-major (<= 2^16 x 2^16 cells = 34 GB,
// the reference's MAX_KERNEL_CELLS cap, inside one B200's HBM).  One sweep is
// two streaming passes over it, both coalesced along j:
//   column pass  kta_j = sum_i K_ij a_i   (a_i = mu_i / kb_i formed on the fly;
//                 row chunks of CH rows write partials, a second kernel folds
//                 them in chunk order and forms b_j = nu_j / kta_j)
//   row pass     kb_i = sum_j K_ij b_j    (one warp per row)
// so a sweep moves 16 * ns * nt bytes: HBM-bound.  Marginal gap, range checks
// and the zero-denominator checks are fused into the passes; per-block
// partials are folded in a fixed order (deterministic).  The iteration runs
// without host round trips: every kernel first reads a device-side state
// record and does nothing once the fit has stopped; the host checks the
// record every few sweeps.
//
// The log-domain iteration (sinkhorn.py:150-178) overwrites the kernel with
// the cost matrix C and runs logsumexp passes of the same shape (max, then
// sum of exp(x - max), as scipy's logsumexp).
//
// Compiled with --fmad=false: costs, quotients and products are rounded as
// the reference's numpy expressions; sums use a different (fixed) order, so
// results agree to rounding (tests: 1e-9 relative on the bounds).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace gdt {

constexpr int EN_CH = 64;        // rows per column-pass chunk
constexpr int EN_T = 256;        // threads per CTA
constexpr double EN_FLOOR = 1e-100, EN_CEIL = 1e100;  // sinkhorn.py:42-43

struct EnState {
    int done;        // 1 once converged, failed or out of sweeps
    int status;      // 0 ok, 1 zero row, 2 zero col, 3 overflow (plain) / non-finite (log)
    int iterations;  // completed sweeps
    int converged;
    double gap;
    double xi;
    int max_iter;
    int pad;
};

__device__ __forceinline__ double en_cost(const double *__restrict__ xs,
                                          const double *__restrict__ xt, int64_t i, int64_t j,
                                          int d, double p) {
    // cdist(sqeuclidean): sum over axes in order, then rho^p (costs.py:44-53)
    double sq = 0.0;
    for (int a = 0; a < d; ++a) {
        const double t = xs[i * d + a] - xt[j * d + a];
        sq = __dadd_rn(sq, __dmul_rn(t, t));
    }
    if (p == 2.0) return sq;
    if (p == 1.0) return sqrt(sq);
    return pow(sq, p / 2.0);
}

// K_ij = exp(-C_ij / eps) (plain) or C_ij (log domain)
__global__ void en_fill_kernel(const double *__restrict__ xs, const double *__restrict__ xt,
                               int64_t ns, int64_t nt, int d, double p, double eps, int gibbs,
                               double *__restrict__ K) {
    const int64_t total = ns * nt;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / nt, j = e - i * nt;
        const double c = en_cost(xs, xt, i, j, d, p);
        K[e] = gibbs ? exp(-c / eps) : c;
    }
}

// deterministic fold of CTA partials: [nb][W] -> out[W] (one CTA)
template <int W>
__device__ void en_block_fold(double (&v)[W], double *sh) {
    // sh: [EN_T][W]
    for (int w = 0; w < W; ++w) sh[threadIdx.x * W + w] = v[w];
    __syncthreads();
    for (int s = EN_T / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
            for (int w = 0; w < W; ++w) {
                // slots 0: sums, 1: min, 2: max (the caller's convention)
                const double o = sh[(threadIdx.x + s) * W + w];
                double &m = sh[threadIdx.x * W + w];
                m = w == 0 ? m + o : (w == 1 ? fmin(m, o) : fmax(m, o));
            }
        __syncthreads();
    }
    for (int w = 0; w < W; ++w) v[w] = sh[w];
}

// ---- plain scaling ---------------------------------------------------------

// row pass: kb_i = sum_j K_ij b_j (one warp per row); with `sweep`, also the
// gap part |a_i kb_i - mu_i| and the positive range of a (block partials)
__global__ void __launch_bounds__(EN_T) en_row_kernel(const double *__restrict__ K,
                                                       const double *__restrict__ b,
                                                       const double *__restrict__ a,
                                                       const double *__restrict__ mu,
                                                       double *__restrict__ kb, int64_t ns,
                                                       int64_t nt, int sweep,
                                                       double *__restrict__ part,
                                                       const EnState *st) {
    __shared__ double sh[EN_T * 3];
    if (st->done) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double v[3] = {0.0, INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * (EN_T / 32) + wib; i < ns;
         i += (int64_t)gridDim.x * (EN_T / 32)) {
        const double *row = K + i * nt;
        // four independent partial sums per lane keep four loads in flight
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int64_t j = lane;
        for (; j + 96 < nt; j += 128) {
            s0 += row[j] * b[j];
            s1 += row[j + 32] * b[j + 32];
            s2 += row[j + 64] * b[j + 64];
            s3 += row[j + 96] * b[j + 96];
        }
        for (; j < nt; j += 32) s0 += row[j] * b[j];
        double s = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            kb[i] = s;
            if (sweep) {
                const double ai = a[i];
                v[0] += fabs(ai * s - mu[i]);
                if (ai > 0.0) {
                    v[1] = fmin(v[1], ai);
                    v[2] = fmax(v[2], ai);
                }
            }
        }
    }
    if (!sweep) return;
    en_block_fold<3>(v, sh);
    if (threadIdx.x == 0)
        for (int w = 0; w < 3; ++w) part[blockIdx.x * 3 + w] = v[w];
}

// column pass: partial[c][j] = sum_{i in chunk c} K_ij a_i with a_i = mu_i / kb_i
// (0 where kb_i <= 0; a zero row with mu_i > 0 raises the row flag);
// CTAs of column-block 0 store a
__global__ void __launch_bounds__(EN_T) en_col_kernel(const double *__restrict__ K,
                                                       const double *__restrict__ kb,
                                                       const double *__restrict__ mu,
                                                       double *__restrict__ a,
                                                       double *__restrict__ partial, int64_t ns,
                                                       int64_t nt, int *flag,
                                                       const EnState *st) {
    __shared__ double as[EN_CH];
    if (st->done) return;
    const int64_t c = blockIdx.y, i0 = c * EN_CH;
    const int rows = (int)std::min<int64_t>(EN_CH, ns - i0);
    for (int r = threadIdx.x; r < rows; r += EN_T) {
        const double k = kb[i0 + r], m = mu[i0 + r];
        const double ai = k > 0.0 ? m / k : 0.0;
        if (k <= 0.0 && m > 0.0) atomicOr(flag, 1);
        as[r] = ai;
        if (blockIdx.x == 0) a[i0 + r] = ai;
    }
    __syncthreads();
    for (int64_t j = blockIdx.x * (int64_t)EN_T + threadIdx.x; j < nt;
         j += (int64_t)gridDim.x * EN_T) {
        double s = 0.0;
        for (int r = 0; r < rows; ++r) s += K[(i0 + r) * nt + j] * as[r];
        partial[c * nt + j] = s;
    }
}

// fold the column partials in chunk order: kta_j, b_j = nu_j / kta_j, the gap
// part |nu_j - b_j kta_j| and the positive range of b (block partials)
__global__ void __launch_bounds__(EN_T) en_colfold_kernel(const double *__restrict__ partial,
                                                           int64_t chunks, const double *__restrict__ nu,
                                                           double *__restrict__ kta,
                                                           double *__restrict__ b, int64_t nt,
                                                           int *flag, double *__restrict__ part,
                                                           const EnState *st) {
    __shared__ double sh[EN_T * 3];
    if (st->done) return;
    double v[3] = {0.0, INFINITY, -INFINITY};
    for (int64_t j = blockIdx.x * (int64_t)EN_T + threadIdx.x; j < nt;
         j += (int64_t)gridDim.x * EN_T) {
        double s = 0.0;
        for (int64_t c = 0; c < chunks; ++c) s += partial[c * nt + j];
        kta[j] = s;
        const double n = nu[j];
        if (s <= 0.0 && n > 0.0) atomicOr(flag, 2);
        const double bj = s > 0.0 ? n / s : 0.0;
        b[j] = bj;
        if (bj > 0.0) {
            v[1] = fmin(v[1], bj);
            v[2] = fmax(v[2], bj);
        }
        // the gap term of b needs kb(b) only for a; nu - b*kta is final here
        v[0] += fabs(n - bj * s);
    }
    en_block_fold<3>(v, sh);
    if (threadIdx.x == 0)
        for (int w = 0; w < 3; ++w) part[blockIdx.x * 3 + w] = v[w];
}

// end of a sweep (one CTA): checks in the reference's order (sinkhorn.py:124-141)
__global__ void en_finish_kernel(const double *__restrict__ rpart, int nr,
                                 const double *__restrict__ cpart, int nc, int *flag,
                                 EnState *st) {
    if (st->done || threadIdx.x != 0) return;
    const int fl = *flag;
    *flag = 0;
    if (fl & 1) { st->status = 1; st->done = 1; return; }
    if (fl & 2) { st->status = 2; st->done = 1; return; }
    double ga = 0.0, lo_a = INFINITY, hi_a = -INFINITY, gb = 0.0, lo_b = INFINITY, hi_b = -INFINITY;
    for (int k = 0; k < nr; ++k) {
        ga += rpart[3 * k];
        lo_a = fmin(lo_a, rpart[3 * k + 1]);
        hi_a = fmax(hi_a, rpart[3 * k + 2]);
    }
    for (int k = 0; k < nc; ++k) {
        gb += cpart[3 * k];
        lo_b = fmin(lo_b, cpart[3 * k + 1]);
        hi_b = fmax(hi_b, cpart[3 * k + 2]);
    }
    st->iterations += 1;
    // _check_scale_range: only positive entries; none -> no check
    const bool bad_a = hi_a >= lo_a && (lo_a < EN_FLOOR || hi_a > EN_CEIL || !isfinite(hi_a));
    const bool bad_b = hi_b >= lo_b && (lo_b < EN_FLOOR || hi_b > EN_CEIL || !isfinite(hi_b));
    if (bad_a || bad_b) { st->status = 3; st->done = 1; return; }
    st->gap = ga + gb;
    if (st->gap < st->xi) { st->converged = 1; st->done = 1; return; }
    if (st->iterations >= st->max_iter) st->done = 1;
}

// ---- log domain ------------------------------------------------------------

// row LSE: out_i = logsumexp_j((g_j - C_ij) / eps) (one warp per row); with
// `sweep`, the gap part |exp(f_i/eps + out_i) - mu_i|
__global__ void __launch_bounds__(EN_T) en_lse_row_kernel(const double *__restrict__ C,
                                                           const double *__restrict__ g,
                                                           const double *__restrict__ f,
                                                           const double *__restrict__ mu,
                                                           double *__restrict__ lkb, int64_t ns,
                                                           int64_t nt, double eps, int sweep,
                                                           double *__restrict__ part,
                                                           const EnState *st) {
    __shared__ double sh[EN_T * 3];
    if (st->done) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double v[3] = {0.0, INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * (EN_T / 32) + wib; i < ns;
         i += (int64_t)gridDim.x * (EN_T / 32)) {
        const double *row = C + i * nt;
        double m = -INFINITY;
        for (int64_t j = lane; j < nt; j += 32) m = fmax(m, (g[j] - row[j]) / eps);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        const double mm = isfinite(m) ? m : 0.0;
        double s = 0.0;
        for (int64_t j = lane; j < nt; j += 32) s += exp((g[j] - row[j]) / eps - mm);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            const double l = log(s) + mm;
            lkb[i] = l;
            if (sweep) v[0] += fabs(exp(f[i] / eps + l) - mu[i]);
        }
    }
    if (!sweep) return;
    en_block_fold<3>(v, sh);
    if (threadIdx.x == 0)
        for (int w = 0; w < 3; ++w) part[blockIdx.x * 3 + w] = v[w];
}

// f_i = eps (log mu_i - lkb_i) for the chunk, then per chunk c the column max
// and the sum of exp(x - max) of x_ij = (f_i - C_ij) / eps
__global__ void __launch_bounds__(EN_T) en_lse_col_kernel(const double *__restrict__ C,
                                                           const double *__restrict__ lkb,
                                                           const double *__restrict__ mu,
                                                           double *__restrict__ f,
                                                           double *__restrict__ pmax,
                                                           double *__restrict__ psum, int64_t ns,
                                                           int64_t nt, double eps,
                                                           const EnState *st) {
    __shared__ double fs[EN_CH];
    if (st->done) return;
    const int64_t c = blockIdx.y, i0 = c * EN_CH;
    const int rows = (int)std::min<int64_t>(EN_CH, ns - i0);
    for (int r = threadIdx.x; r < rows; r += EN_T) {
        const double fi = eps * (log(mu[i0 + r]) - lkb[i0 + r]);
        fs[r] = fi;
        if (blockIdx.x == 0) f[i0 + r] = fi;
    }
    __syncthreads();
    for (int64_t j = blockIdx.x * (int64_t)EN_T + threadIdx.x; j < nt;
         j += (int64_t)gridDim.x * EN_T) {
        double m = -INFINITY;
        for (int r = 0; r < rows; ++r) m = fmax(m, (fs[r] - C[(i0 + r) * nt + j]) / eps);
        double s = 0.0;
        if (isfinite(m))
            for (int r = 0; r < rows; ++r) s += exp((fs[r] - C[(i0 + r) * nt + j]) / eps - m);
        pmax[c * nt + j] = m;
        psum[c * nt + j] = s;
    }
}

// combine the chunks: lkta_j, g_j = eps (log nu_j - lkta_j), gap part
// |nu_j - exp(g_j/eps + lkta_j)|
__global__ void __launch_bounds__(EN_T) en_lse_colfold_kernel(const double *__restrict__ pmax,
                                                               const double *__restrict__ psum,
                                                               int64_t chunks,
                                                               const double *__restrict__ nu,
                                                               double *__restrict__ lkta,
                                                               double *__restrict__ g, int64_t nt,
                                                               double eps, double *__restrict__ part,
                                                               const EnState *st) {
    __shared__ double sh[EN_T * 3];
    if (st->done) return;
    double v[3] = {0.0, INFINITY, -INFINITY};
    for (int64_t j = blockIdx.x * (int64_t)EN_T + threadIdx.x; j < nt;
         j += (int64_t)gridDim.x * EN_T) {
        double M = -INFINITY;
        for (int64_t c = 0; c < chunks; ++c) M = fmax(M, pmax[c * nt + j]);
        const double mm = isfinite(M) ? M : 0.0;
        double s = 0.0;
        for (int64_t c = 0; c < chunks; ++c) {
            const double m = pmax[c * nt + j];
            if (isfinite(m)) s += psum[c * nt + j] * exp(m - mm);
        }
        const double l = log(s) + mm;
        lkta[j] = l;
        const double gj = eps * (log(nu[j]) - l);
        g[j] = gj;
        v[0] += fabs(nu[j] - exp(gj / eps + l));
    }
    en_block_fold<3>(v, sh);
    if (threadIdx.x == 0)
        for (int w = 0; w < 3; ++w) part[blockIdx.x * 3 + w] = v[w];
}

__global__ void en_lse_finish_kernel(const double *__restrict__ rpart, int nr,
                                     const double *__restrict__ cpart, int nc, EnState *st) {
    if (st->done || threadIdx.x != 0) return;
    double ga = 0.0, gb = 0.0;
    for (int k = 0; k < nr; ++k) ga += rpart[3 * k];
    for (int k = 0; k < nc; ++k) gb += cpart[3 * k];
    st->iterations += 1;
    st->gap = ga + gb;
    if (st->gap < st->xi) { st->converged = 1; st->done = 1; return; }
    if (st->iterations >= st->max_iter) st->done = 1;
}

// f = eps log a, g = eps log b after a successful plain fit (sinkhorn.py:187-189)
__global__ void en_log_kernel(const double *__restrict__ x, double *__restrict__ out, int64_t n,
                              double eps) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = eps * log(x[i]);
}

__global__ void en_finite_kernel(const double *__restrict__ x, int64_t n, int *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) atomicOr(bad, 1);
}

// ---- plan pricing (sinkhorn.py:268-276) ------------------------------------

// P_ij = exp((f_i + g_j - C_ij) / eps): row sums (warp per row), per-row
// transport sums, column partials per row chunk
__global__ void __launch_bounds__(EN_T) en_plan_row_kernel(
    const double *__restrict__ xs, const double *__restrict__ xt, int64_t ns, int64_t nt, int d,
    double p, double eps, const double *__restrict__ f, const double *__restrict__ g,
    double *__restrict__ mu_hat, double *__restrict__ trow) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int64_t i = (int64_t)blockIdx.x * (EN_T / 32) + wib; i < ns;
         i += (int64_t)gridDim.x * (EN_T / 32)) {
        double s = 0.0, t = 0.0;
        for (int64_t j = lane; j < nt; j += 32) {
            const double c = en_cost(xs, xt, i, j, d, p);
            const double pl = exp((f[i] + g[j] - c) / eps);
            s += pl;
            t += pl * c;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            t += __shfl_xor_sync(0xffffffffu, t, o);
        }
        if (lane == 0) {
            mu_hat[i] = s;
            trow[i] = t;
        }
    }
}

__global__ void __launch_bounds__(EN_T) en_plan_col_kernel(
    const double *__restrict__ xs, const double *__restrict__ xt, int64_t ns, int64_t nt, int d,
    double p, double eps, const double *__restrict__ f, const double *__restrict__ g,
    double *__restrict__ partial) {
    const int64_t c = blockIdx.y, i0 = c * EN_CH;
    const int rows = (int)std::min<int64_t>(EN_CH, ns - i0);
    for (int64_t j = blockIdx.x * (int64_t)EN_T + threadIdx.x; j < nt;
         j += (int64_t)gridDim.x * EN_T) {
        double s = 0.0;
        for (int r = 0; r < rows; ++r) {
            const double cst = en_cost(xs, xt, i0 + r, j, d, p);
            s += exp((f[i0 + r] + g[j] - cst) / eps);
        }
        partial[c * nt + j] = s;
    }
}

__global__ void en_plan_fold_kernel(const double *__restrict__ partial, int64_t chunks,
                                    double *__restrict__ nu_hat, int64_t nt,
                                    const double *__restrict__ trow, int64_t ns,
                                    double *__restrict__ total) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nt;
         j += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t c = 0; c < chunks; ++c) s += partial[c * nt + j];
        nu_hat[j] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double t = 0.0;
        for (int64_t i = 0; i < ns; ++i) t += trow[i];
        *total = t;
    }
}

// ---- host driver --------------------------------------------------------------

struct EnLayout {
    int64_t chunks, rblocks, cblocks, colx;
    size_t off_state, off_flag, off_a, off_b, off_kb, off_kta, off_part, off_part2, off_rpart,
        off_cpart, off_K, total;
};

static EnLayout en_layout(int64_t ns, int64_t nt) {
    EnLayout L;
    L.chunks = (ns + EN_CH - 1) / EN_CH;
    L.rblocks = std::min<int64_t>((ns + EN_T / 32 - 1) / (EN_T / 32), 148 * 8);
    L.cblocks = std::min<int64_t>((nt + EN_T - 1) / EN_T, 148 * 8);
    L.colx = std::min<int64_t>((nt + EN_T - 1) / EN_T, 64);
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o += (bytes + 255) & ~(size_t)255;
        return at;
    };
    L.off_state = take(sizeof(EnState));
    L.off_flag = take(sizeof(int) * 2);
    L.off_a = take(sizeof(double) * ns);
    L.off_b = take(sizeof(double) * nt);
    L.off_kb = take(sizeof(double) * ns);
    L.off_kta = take(sizeof(double) * nt);
    L.off_part = take(sizeof(double) * L.chunks * nt);
    L.off_part2 = take(sizeof(double) * L.chunks * nt);
    L.off_rpart = take(sizeof(double) * 3 * L.rblocks);
    L.off_cpart = take(sizeof(double) * 3 * L.cblocks);
    L.off_K = take(sizeof(double) * ns * nt);
    L.total = o;
    return L;
}

}  // namespace gdt

using namespace gdt;

extern "C" int64_t gdt_entropic_scratch_bytes(int64_t ns, int64_t nt) {
    if (ns < 1 || nt < 1) return 0;
    return (int64_t)en_layout(ns, nt).total;
}

extern "C" int gdt_entropic_fit(const double *xs, const double *xt, int64_t ns, int64_t nt,
                                int d, double p, double eps, const double *mu, const double *nu,
                                double xi, int64_t max_iter, double *f, double *g, double *info,
                                int32_t *status, void *scratch, void *stream) {
    GDT_CHECK_ARG(ns >= 1 && nt >= 1 && d >= 1 && p >= 1.0 && eps > 0.0 && max_iter >= 1 &&
                      max_iter < (1ll << 31) && scratch != nullptr,
                  "gdt_entropic_fit: bad arguments");
    cudaStream_t st = as_stream(stream);
    const EnLayout L = en_layout(ns, nt);
    char *base = static_cast<char *>(scratch);
    EnState *S = reinterpret_cast<EnState *>(base + L.off_state);
    int *flag = reinterpret_cast<int *>(base + L.off_flag);
    double *a = reinterpret_cast<double *>(base + L.off_a);
    double *b = reinterpret_cast<double *>(base + L.off_b);
    double *kb = reinterpret_cast<double *>(base + L.off_kb);
    double *kta = reinterpret_cast<double *>(base + L.off_kta);
    double *part = reinterpret_cast<double *>(base + L.off_part);
    double *part2 = reinterpret_cast<double *>(base + L.off_part2);
    double *rpart = reinterpret_cast<double *>(base + L.off_rpart);
    double *cpart = reinterpret_cast<double *>(base + L.off_cpart);
    double *K = reinterpret_cast<double *>(base + L.off_K);
    const dim3 cgrid((unsigned)L.colx, (unsigned)L.chunks);

    auto reset = [&](EnState &h) -> int {
        h = EnState{0, 0, 0, 0, INFINITY, xi, (int)max_iter, 0};
        if (cudaMemcpyAsync(S, &h, sizeof(EnState), cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaMemsetAsync(flag, 0, sizeof(int) * 2, st) != cudaSuccess)
            return cuda_status("gdt_entropic_fit: state");
        return GDT_OK;
    };
    // run sweeps until the device state says stop; checks the state every
    // `chunk` sweeps (growing), so the stream is not drained every sweep
    auto drive = [&](auto sweep, EnState &h) -> int {
        int64_t issued = 0, chunk = 4;
        for (;;) {
            for (int64_t k = 0; k < chunk && issued < max_iter; ++k, ++issued) sweep();
            if (cudaMemcpyAsync(&h, S, sizeof(EnState), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                return cuda_status("gdt_entropic_fit: sweep");
            if (h.done || issued >= max_iter) return GDT_OK;
            chunk = std::min<int64_t>(chunk * 2, 256);
        }
    };

    // plain scaling on K = exp(-C / eps) (ipf_fit, sinkhorn.py:101-142)
    EnState h;
    if (int rc = reset(h)) return rc;
    en_fill_kernel<<<grid_size(ns * nt, 256), 256, 0, st>>>(xs, xt, ns, nt, d, p, eps, 1, K);
    std::vector<double> ones(nt, 1.0);
    cudaMemcpyAsync(b, ones.data(), sizeof(double) * nt, cudaMemcpyHostToDevice, st);
    en_row_kernel<<<(unsigned)L.rblocks, EN_T, 0, st>>>(K, b, a, mu, kb, ns, nt, 0, rpart, S);
    auto plain_sweep = [&]() {
        en_col_kernel<<<cgrid, EN_T, 0, st>>>(K, kb, mu, a, part, ns, nt, flag, S);
        en_colfold_kernel<<<(unsigned)L.cblocks, EN_T, 0, st>>>(part, L.chunks, nu, kta, b, nt,
                                                                 flag, cpart, S);
        en_row_kernel<<<(unsigned)L.rblocks, EN_T, 0, st>>>(K, b, a, mu, kb, ns, nt, 1, rpart, S);
        en_finish_kernel<<<1, 32, 0, st>>>(rpart, (int)L.rblocks, cpart, (int)L.cblocks, flag, S);
    };
    if (int rc = cuda_status("gdt_entropic_fit: setup")) return rc;
    if (int rc = drive(plain_sweep, h)) return rc;
    int log_domain = 0;
    if (h.status == 0) {
        en_log_kernel<<<grid_size(ns, 256), 256, 0, st>>>(a, f, ns, eps);
        en_log_kernel<<<grid_size(nt, 256), 256, 0, st>>>(b, g, nt, eps);
    } else {
        // zero denominator or scale overflow: restart in the log domain
        // (_run_scaling, sinkhorn.py:181-195; _log_domain_scaling :150-178)
        log_domain = 1;
        if (int rc = reset(h)) return rc;
        en_fill_kernel<<<grid_size(ns * nt, 256), 256, 0, st>>>(xs, xt, ns, nt, d, p, eps, 0, K);
        cudaMemsetAsync(g, 0, sizeof(double) * nt, st);
        en_lse_row_kernel<<<(unsigned)L.rblocks, EN_T, 0, st>>>(K, g, f, mu, kb, ns, nt, eps, 0,
                                                                 rpart, S);
        auto log_sweep = [&]() {
            en_lse_col_kernel<<<cgrid, EN_T, 0, st>>>(K, kb, mu, f, part, part2, ns, nt, eps, S);
            en_lse_colfold_kernel<<<(unsigned)L.cblocks, EN_T, 0, st>>>(part, part2, L.chunks, nu,
                                                                         kta, g, nt, eps, cpart, S);
            en_lse_row_kernel<<<(unsigned)L.rblocks, EN_T, 0, st>>>(K, g, f, mu, kb, ns, nt, eps, 1,
                                                                     rpart, S);
            en_lse_finish_kernel<<<1, 32, 0, st>>>(rpart, (int)L.rblocks, cpart, (int)L.cblocks, S);
        };
        if (int rc = drive(log_sweep, h)) return rc;
        en_finite_kernel<<<grid_size(ns, 256), 256, 0, st>>>(f, ns, flag);
        en_finite_kernel<<<grid_size(nt, 256), 256, 0, st>>>(g, nt, flag);
        int bad = 0;
        cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_status("gdt_entropic_fit: log");
        h.status = bad ? 3 : 0;
    }
    const double host_info[4] = {(double)h.iterations, h.gap, (double)h.converged,
                                 (double)log_domain};
    const int32_t s32 = h.status == 0 ? GDT_PAIR_OK : GDT_PAIR_OVERFLOW;
    cudaMemcpyAsync(info, host_info, sizeof(host_info), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(status, &s32, sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_status("gdt_entropic_fit: out");
    return cuda_status("gdt_entropic_fit");
}

extern "C" int gdt_entropic_plan(const double *xs, const double *xt, int64_t ns, int64_t nt,
                                 int d, double p, double eps, const double *f, const double *g,
                                 double *mu_hat, double *nu_hat, double *transport,
                                 void *scratch, void *stream) {
    GDT_CHECK_ARG(ns >= 1 && nt >= 1 && d >= 1 && p >= 1.0 && eps > 0.0 && scratch != nullptr,
                  "gdt_entropic_plan: bad arguments");
    cudaStream_t st = as_stream(stream);
    const EnLayout L = en_layout(ns, nt);
    char *base = static_cast<char *>(scratch);
    double *part = reinterpret_cast<double *>(base + L.off_part);
    double *trow = reinterpret_cast<double *>(base + L.off_kb);
    en_plan_row_kernel<<<(unsigned)L.rblocks, EN_T, 0, st>>>(xs, xt, ns, nt, d, p, eps, f, g,
                                                             mu_hat, trow);
    en_plan_col_kernel<<<dim3((unsigned)L.colx, (unsigned)L.chunks), EN_T, 0, st>>>(
        xs, xt, ns, nt, d, p, eps, f, g, part);
    en_plan_fold_kernel<<<grid_size(nt, 256), 256, 0, st>>>(part, L.chunks, nu_hat, nt, trow, ns,
                                                           transport);
    return cuda_status("gdt_entropic_plan");
}
