// Grid primitives: padding, SumPool (K1), potential interpolation (K8),
// coarse c-transform (K7), weighted-TV inner sums and batched dots (K10).
// Compiled with --fmad=false: every expression here is rounded exactly as
// the reference's numpy expression it restates.
#include <cstdio>
#include <mutex>
#include <string>

#include <algorithm>

#include "common.cuh"

namespace gdt {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

// Stream-ordered workspaces come from the device's default memory pool; keep
// freed blocks cached in the pool (release threshold = max) so repeated calls
// do not map and unmap device memory at every synchronisation.
cudaError_t malloc_async(void **p, size_t bytes, cudaStream_t st) {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev != done_dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        done_dev = dev;
    }
    return cudaMallocAsync(p, bytes, st);
}

int cuda_status(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(where) + ": " + cudaGetErrorString(e));
        return GDT_ERR_CUDA;
    }
    return GDT_OK;
}

// ---------------------------------------------------------------------------
// padding (measures.py:236-245)
// ---------------------------------------------------------------------------
__global__ void pad_kernel(const double *__restrict__ in, double *__restrict__ out,
                           int64_t batch, Grid src, Grid dst) {
    const int64_t total = batch * dst.cells;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / dst.cells;
        int64_t rem = idx - b * dst.cells;
        int64_t src_off = 0;
        bool inside = true;
        for (int a = dst.nd - 1; a >= 0; --a) {
            const int64_t x = rem / dst.stride[a];
            rem -= x * dst.stride[a];
            if (x >= src.n[a]) inside = false;
            src_off += x * src.stride[a];
        }
        out[idx] = inside ? in[b * src.cells + src_off] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// K1 SumPool: one thread per (pair, block); offsets visited in ascending fine
// flat order, accumulator starts at 0.0 (np.add.at order, measures.py:266).
// ---------------------------------------------------------------------------
// With `stats`, the same pass also records per block the smallest and largest
// positive mass and the number of positive cells ([batch, n, 3]; +inf / -inf /
// 0 for a block without support) -- the block statistics of the coarse-level
// primal stage (primal.cu), at no extra read of the fine masses.
__global__ void sumpool_kernel(const double *__restrict__ fine, double *__restrict__ coarse,
                               int64_t batch, Grid f, Grid c, int kappa,
                               double *__restrict__ stats) {
    const int64_t total = batch * c.cells;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / c.cells;
        int64_t rem = idx - b * c.cells;
        int64_t origin = 0;
        for (int a = c.nd - 1; a >= 0; --a) {
            const int64_t x = rem / c.stride[a];
            rem -= x * c.stride[a];
            origin += x * kappa * f.stride[a];
        }
        const double *src = fine + b * f.cells + origin;
        const int K3 = c.nd > 3 ? kappa : 1, K2 = c.nd > 2 ? kappa : 1, K1 = c.nd > 1 ? kappa : 1;
        double acc = 0.0, lo = INFINITY, hi = -INFINITY, cnt = 0.0;
        for (int o3 = 0; o3 < K3; ++o3)
            for (int o2 = 0; o2 < K2; ++o2)
                for (int o1 = 0; o1 < K1; ++o1) {
                    const double *row = src + o3 * f.stride[3] + o2 * f.stride[2] + o1 * f.stride[1];
                    for (int o0 = 0; o0 < kappa; ++o0) {
                        const double x = row[o0];
                        acc = __dadd_rn(acc, x);
                        if (x > 0.0) {
                            lo = fmin(lo, x);
                            hi = fmax(hi, x);
                            cnt += 1.0;
                        }
                    }
                }
        coarse[idx] = acc;
        if (stats) {
            stats[3 * idx] = lo;
            stats[3 * idx + 1] = hi;
            stats[3 * idx + 2] = cnt;
        }
    }
}

// ---------------------------------------------------------------------------
// K8 interpolation (quantized.py:388-447).  `axes` holds the sorted coarse
// axis values (np.unique of the centre columns) of every axis back to back.
// i0 = clip(searchsorted(ax, q, 'right') - 1, 0, n-2), t = (q - c_i0) / span
// rounded once and clipped to [0,1]; corners in itertools.product order (last
// axis fastest), weights multiplied in axis order from 1.0, accumulated from
// 0.0.  "nearest" = searchsorted(midpoints, q, 'left').
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t upper_count(const double *ax, int64_t n, double q) {
    int64_t lo = 0, hi = n;  // number of ax[j] <= q
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ax[mid] <= q) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Multilinear interpolation with the per-axis bracket (lo, hi, t) of every
// fine coordinate precomputed once per CTA in shared memory (the same
// arithmetic as interpolate_kernel, which recomputes it per cell).
constexpr int IP_MAX_AX = 2048;  // sum of fine axis lengths handled by the table kernel

template <int ND>  // compile-time dimension (0: runtime): corner loop fully unrolled
__global__ void __launch_bounds__(256) interpolate_tab_kernel(
    const double *__restrict__ coarse, double *__restrict__ fine, int64_t batch, Grid f, Grid c,
    const double *__restrict__ axes) {
    __shared__ double tt_s[IP_MAX_AX];
    __shared__ int lo_s[IP_MAX_AX], hi_s[IP_MAX_AX];
    int base[GDT_MAX_DIM], cb[GDT_MAX_DIM];
    {
        int o = 0, co = 0;
        for (int a = 0; a < f.nd; ++a) {
            base[a] = o;
            cb[a] = co;
            o += (int)f.n[a];
            co += (int)c.n[a];
        }
        for (int e = threadIdx.x; e < o; e += blockDim.x) {
            int a = 0;
            while (a + 1 < f.nd && e >= base[a + 1]) ++a;
            const double q = (double)(e - base[a] + 1);  // 1-based coordinate
            const double *ax = axes + cb[a];
            const int64_t n = c.n[a];
            int64_t i0 = upper_count(ax, n, q) - 1;
            const int64_t top = n - 2 > 0 ? n - 2 : 0;
            if (i0 < 0) i0 = 0;
            if (i0 > top) i0 = top;
            const int64_t i1 = i0 + 1 < n - 1 ? i0 + 1 : n - 1;
            const double span = __dsub_rn(ax[i1], ax[i0]);
            double t = span > 0.0 ? __ddiv_rn(__dsub_rn(q, ax[i0]), span) : 0.0;
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
            lo_s[e] = (int)i0;
            hi_s[e] = (int)i1;
            tt_s[e] = t;
        }
    }
    __syncthreads();
    const int64_t total = batch * f.cells;
    const int nd = ND ? ND : f.nd;
    int fs[GDT_MAX_DIM], cs[GDT_MAX_DIM];
#pragma unroll
    for (int a = 0; a < GDT_MAX_DIM; ++a) {
        fs[a] = (int)f.stride[a];
        cs[a] = (int)c.stride[a];
    }
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / f.cells;
        int rem = (int)(idx - b * f.cells);
        // per axis, once per cell: both weights and both coarse offsets
        double wt[GDT_MAX_DIM][2];
        int of[GDT_MAX_DIM][2];
#pragma unroll
        for (int a = GDT_MAX_DIM - 1; a >= 0; --a)
            if (a < nd) {
                const int x = rem / fs[a];
                rem -= x * fs[a];
                const int e = base[a] + x;
                const double t = tt_s[e];
                wt[a][0] = __dsub_rn(1.0, t);
                wt[a][1] = t;
                of[a][0] = lo_s[e] * cs[a];
                of[a][1] = hi_s[e] * cs[a];
            }
        const double *T = coarse + b * c.cells;
        double out = 0.0;
        // corners in the reference's order (axis 0 slowest); the weight is the
        // left-to-right product 1 * w_0 * w_1 * ... (1 * w_0 is exact)
#pragma unroll
        for (int cidx = 0; cidx < (1 << (ND ? ND : GDT_MAX_DIM)); ++cidx) {
            if (cidx >= (1 << nd)) break;
            double w = 1.0;
            int off = 0;
#pragma unroll
            for (int a = 0; a < GDT_MAX_DIM; ++a)
                if (a < nd) {
                    const int side = (cidx >> (nd - 1 - a)) & 1;
                    w = a == 0 ? wt[0][side] : __dmul_rn(w, wt[a][side]);
                    off += of[a][side];
                }
            out = __dadd_rn(out, __dmul_rn(w, __ldg(T + off)));
        }
        fine[idx] = out;
    }
}

__global__ void interpolate_kernel(const double *__restrict__ coarse, double *__restrict__ fine,
                                   int64_t batch, Grid f, Grid c, const double *__restrict__ axes,
                                   int method) {
    const int64_t total = batch * f.cells;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / f.cells;
        int64_t rem = idx - b * f.cells;
        double q[GDT_MAX_DIM];
        for (int a = f.nd - 1; a >= 0; --a) {
            const int64_t x = rem / f.stride[a];
            rem -= x * f.stride[a];
            q[a] = (double)(x + 1);  // 1-based coordinate
        }
        const double *T = coarse + b * c.cells;
        if (method == 1) {
            int64_t off = 0, a0 = 0;
            for (int a = 0; a < f.nd; ++a) {
                const double *ax = axes + a0;
                const int64_t n = c.n[a];
                int64_t lo = 0, hi = n - 1;  // midpoints strictly below q
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    const double mp = __ddiv_rn(__dadd_rn(ax[mid], ax[mid + 1]), 2.0);
                    if (mp < q[a]) lo = mid + 1;
                    else hi = mid;
                }
                off += lo * c.stride[a];
                a0 += n;
            }
            fine[idx] = T[off];
            continue;
        }
        int64_t lo[GDT_MAX_DIM], hi[GDT_MAX_DIM];
        double t[GDT_MAX_DIM];
        int64_t a0 = 0;
        for (int a = 0; a < f.nd; ++a) {
            const double *ax = axes + a0;
            const int64_t n = c.n[a];
            a0 += n;
            int64_t i0 = upper_count(ax, n, q[a]) - 1;
            const int64_t top = n - 2 > 0 ? n - 2 : 0;
            if (i0 < 0) i0 = 0;
            if (i0 > top) i0 = top;
            const int64_t i1 = i0 + 1 < n - 1 ? i0 + 1 : n - 1;
            const double span = __dsub_rn(ax[i1], ax[i0]);
            double tt = span > 0.0 ? __ddiv_rn(__dsub_rn(q[a], ax[i0]), span) : 0.0;
            tt = tt < 0.0 ? 0.0 : (tt > 1.0 ? 1.0 : tt);
            lo[a] = i0;
            hi[a] = i1;
            t[a] = tt;
        }
        double out = 0.0;
        const int corners = 1 << f.nd;
        for (int cidx = 0; cidx < corners; ++cidx) {
            double w = 1.0;
            int64_t off = 0;
            for (int a = 0; a < f.nd; ++a) {
                const int side = (cidx >> (f.nd - 1 - a)) & 1;  // axis 0 slowest
                w = __dmul_rn(w, side ? t[a] : __dsub_rn(1.0, t[a]));
                off += (side ? hi[a] : lo[a]) * c.stride[a];
            }
            out = __dadd_rn(out, __dmul_rn(w, T[off]));
        }
        fine[idx] = out;
    }
}

// ---------------------------------------------------------------------------
// K7 coarse c-transform over the coarse target support (quantized.py:504-505)
// ---------------------------------------------------------------------------
// one warp per (pair, k): lanes stride over the target support (coalesced
// reads of the C-tilde row), exact min reduced across the warp
__global__ void __launch_bounds__(256) coarse_ct_kernel(const double *__restrict__ g,
                                                        const int32_t *__restrict__ dst,
                                                        const int32_t *__restrict__ supp_len,
                                                        const double *__restrict__ C, int64_t n,
                                                        int64_t batch, double *__restrict__ f_ext) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= batch * n) return;
    const int64_t b = w / n, k = w - b * n;
    const int len = supp_len[b];
    const double *gb = g + b * n;
    const int32_t *db = dst + b * n;
    const double *Ck = C + k * n;
    double best = INFINITY;
    if (len == n) {  // full target support: dst is the identity, the row is contiguous
        int l = lane;
        double b1 = INFINITY;
        for (; l + 32 < len; l += 64) {
            best = fmin(best, __dsub_rn(__ldg(Ck + l), __ldg(gb + l)));
            b1 = fmin(b1, __dsub_rn(__ldg(Ck + l + 32), __ldg(gb + l + 32)));
        }
        for (; l < len; l += 32) best = fmin(best, __dsub_rn(__ldg(Ck + l), __ldg(gb + l)));
        best = fmin(best, b1);
    } else {
        for (int l = lane; l < len; l += 32) best = fmin(best, __dsub_rn(Ck[db[l]], gb[l]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) f_ext[w] = best;
}

// ---------------------------------------------------------------------------
// weighted-TV inner sums (measures.py:289-315, before the 1/p root) and
// batched dots: block-per-pair fp64 reductions (BLAS-like, any order).
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) tv_inner_kernel(const double *__restrict__ x,
                                                           const double *__restrict__ y,
                                                           Grid g, double p,
                                                           const double *__restrict__ wts,
                                                           double *__restrict__ out) {
    __shared__ double sh[32];
    const int64_t b = blockIdx.x;
    const double *xb = x + b * g.cells, *yb = y + b * g.cells;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < g.cells; i += THREADS) {
        int64_t rem = i;
        double sq = -0.0;
        double parts[GDT_MAX_DIM];
        for (int a = g.nd - 1; a >= 0; --a) {
            const int64_t xa = rem / g.stride[a];
            rem -= xa * g.stride[a];
            const double ctr = ((double)g.n[a] + 1.0) / 2.0;
            const double df = __dsub_rn((double)(xa + 1), ctr);
            parts[a] = __dmul_rn(df, df);
        }
        for (int a = 0; a < g.nd; ++a) sq = __dadd_rn(sq, parts[a]);
        double w;
        if (wts != nullptr) w = wts[i];
        else if (p == 2.0) w = sq;
        else if (p == 1.0) w = __dsqrt_rn(sq);
        else w = pow(sq, p / 2.0);
        acc += __dmul_rn(w, fabs(__dsub_rn(xb[i], yb[i])));
    }
    acc = block_sum<THREADS>(acc, sh);
    if (threadIdx.x == 0) out[b] = acc;
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) dot_kernel(const double *__restrict__ a,
                                                      const double *__restrict__ bv, int64_t n,
                                                      double *__restrict__ out) {
    __shared__ double sh[32];
    const int64_t b = blockIdx.x;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += THREADS) acc += __dmul_rn(a[b * n + i], bv[b * n + i]);
    acc = block_sum<THREADS>(acc, sh);
    if (threadIdx.x == 0) out[b] = acc;
}

}  // namespace gdt

using namespace gdt;

extern "C" {

const char *gdt_version(void) { return "gridot_b200 0.1.0 (sm_100a)"; }

const char *gdt_last_error(void) { return g_last_error.c_str(); }

int gdt_pad_f64(const double *in, double *out, int64_t batch, int ndim, const int64_t *dims,
                int kappa, void *stream) {
    Grid s, d;
    GDT_CHECK_ARG(make_grid(s, ndim, dims) && kappa >= 1 && batch >= 0, "gdt_pad_f64: bad grid");
    int64_t pd[GDT_MAX_DIM];
    for (int a = 0; a < ndim; ++a) pd[a] = kappa * ((dims[a] + kappa - 1) / kappa);
    make_grid(d, ndim, pd);
    if (batch == 0) return GDT_OK;
    pad_kernel<<<grid_size(batch * d.cells, 256) > 4096 ? 4096 : grid_size(batch * d.cells, 256), 256, 0,
                 as_stream(stream)>>>(in, out, batch, s, d);
    return cuda_status("gdt_pad_f64");
}

int gdt_sumpool_f64(const double *fine, double *coarse, int64_t batch, int ndim,
                    const int64_t *dims, int kappa, void *stream) {
    return gdt_sumpool_stats_f64(fine, coarse, nullptr, batch, ndim, dims, kappa, stream);
}

int gdt_sumpool_stats_f64(const double *fine, double *coarse, double *stats, int64_t batch,
                          int ndim, const int64_t *dims, int kappa, void *stream) {
    Grid f, c;
    GDT_CHECK_ARG(make_grid(f, ndim, dims) && make_coarse(c, f, kappa) && batch >= 0,
                  "gdt_sumpool_f64: dims must be positive multiples of kappa");
    if (batch == 0) return GDT_OK;
    const int64_t work = batch * c.cells;
    sumpool_kernel<<<grid_size(work, 128), 128, 0, as_stream(stream)>>>(fine, coarse, batch, f, c,
                                                                        kappa, stats);
    return cuda_status("gdt_sumpool_f64");
}

int gdt_interpolate(const double *coarse, double *fine, int64_t batch, int ndim,
                    const int64_t *dims, const int64_t *cdims, const double *axes, int method,
                    void *stream) {
    Grid f, c;
    GDT_CHECK_ARG(make_grid(f, ndim, dims) && make_grid(c, ndim, cdims) && axes != nullptr,
                  "gdt_interpolate: bad grid");
    GDT_CHECK_ARG(method == 0 || method == 1, "gdt_interpolate: method must be 0 or 1");
    if (batch == 0) return GDT_OK;
    int64_t axsum = 0;
    for (int a = 0; a < ndim; ++a) axsum += dims[a];
    if (method == 0 && axsum <= IP_MAX_AX && f.cells < (1ll << 31)) {
        const int64_t want = (batch * f.cells + 255) / 256;
        const unsigned ctas = (unsigned)std::min<int64_t>(want, 148 * 8);  // amortise the tables
        if (ndim == 2)
            interpolate_tab_kernel<2><<<ctas, 256, 0, as_stream(stream)>>>(coarse, fine, batch, f, c, axes);
        else if (ndim == 3)
            interpolate_tab_kernel<3><<<ctas, 256, 0, as_stream(stream)>>>(coarse, fine, batch, f, c, axes);
        else
            interpolate_tab_kernel<0><<<ctas, 256, 0, as_stream(stream)>>>(coarse, fine, batch, f, c, axes);
    } else {
        interpolate_kernel<<<grid_size(batch * f.cells, 256), 256, 0, as_stream(stream)>>>(
            coarse, fine, batch, f, c, axes, method);
    }
    return cuda_status("gdt_interpolate");
}

int gdt_coarse_ctransform(const double *g, const int32_t *dst, const int32_t *supp_len,
                          const double *centre_cost, int64_t n, int64_t batch, double *f_ext,
                          void *stream) {
    GDT_CHECK_ARG(n >= 1 && batch >= 0, "gdt_coarse_ctransform: bad sizes");
    if (batch == 0) return GDT_OK;
    coarse_ct_kernel<<<grid_size(batch * n * 32, 256), 256, 0, as_stream(stream)>>>(
        g, dst, supp_len, centre_cost, n, batch, f_ext);
    return cuda_status("gdt_coarse_ctransform");
}

int gdt_weighted_tv_inner(const double *x, const double *y, int64_t batch, int ndim,
                          const int64_t *dims, double p, const double *weights, double *out,
                          void *stream) {
    Grid g;
    GDT_CHECK_ARG(make_grid(g, ndim, dims) && p >= 1.0, "gdt_weighted_tv_inner: bad args");
    if (batch == 0) return GDT_OK;
    tv_inner_kernel<256><<<(unsigned)batch, 256, 0, as_stream(stream)>>>(x, y, g, p, weights,
                                                                             out);
    return cuda_status("gdt_weighted_tv_inner");
}

int gdt_batched_dot(const double *a, const double *b, int64_t batch, int64_t n, double *out,
                    void *stream) {
    GDT_CHECK_ARG(batch >= 0 && n >= 0, "gdt_batched_dot: bad sizes");
    if (batch == 0) return GDT_OK;
    dot_kernel<256><<<(unsigned)batch, 256, 0, as_stream(stream)>>>(a, b, n, out);
    return cuda_status("gdt_batched_dot");
}

}  // extern "C"
