// K9/K10: c-transforms on the fine grid and the fused dual dot.
//
// Reference: c_transform (quantized.py:450-484) evaluates
//   out_j = min_i rho(x_i, x_j)^p - v_i
// brute force over cost blocks of 1024 outputs; dual_upscaling_lower_bound
// applies it twice on one grid (quantized.py:510-511).  Every candidate is
// rounded once and the min is exact, so any evaluation order gives the same
// fp64 result.
//
// p == 2: the grid cost is separable, sum_a (x_a - y_a)^2, so the transform is
// d successive 1-D min-plus passes (O(d N^{d+1}) instead of O(N^{2d})).  For
// the dyadic potentials of the bounds (kappa a power of two) every
// intermediate is exact and the result equals the brute force bit for bit.
// p != 2: tiled brute force.  A thread owns R consecutive outputs along axis
// 0; sources stream through shared memory in rows, and because the cost only
// depends on (dx, dy) the R x S candidate block of a source row needs only
// R + S - 1 distinct costs (Toeplitz reuse).  fp32 uses packed FADD2 + the
// 3-input FMNMX3 of sm_100 (one instruction per candidate).
#include "common.cuh"

namespace gdt {

// ---------------------------------------------------------------------------
// separable p == 2: one pass along axis `ax`
//   out[.., j, ..] = min_i (i - j)^2 + sign * in[.., i, ..]
// ---------------------------------------------------------------------------
// Register-tiled 1-D min-plus pass (the same arithmetic as sep_pass_kernel:
// cand = (TO)(d*d) + line[i], exact min): a thread owns 8 consecutive outputs
// of one line and sweeps the sources 8 at a time; the 15 squared offsets of a
// chunk come from a shared table (aligned 16-byte reads) and fp32 candidates
// use packed add.f32x2 + 3-input min.  Lines of the CTA are interleaved so
// strided-axis loads and stores coalesce.
__device__ __forceinline__ void add_f32x2(float c0, float c1, float v0, float v1, float &r0,
                                          float &r1) {
    unsigned long long rr;
    asm("add.rn.f32x2 %0, %1, %2;"
        : "=l"(rr)
        : "l"((unsigned long long)__float_as_uint(c0) | ((unsigned long long)__float_as_uint(c1) << 32)),
          "l"((unsigned long long)__float_as_uint(v0) | ((unsigned long long)__float_as_uint(v1) << 32)));
    r0 = __uint_as_float((unsigned)(rr & 0xffffffffu));
    r1 = __uint_as_float((unsigned)(rr >> 32));
}

__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

constexpr int SEPT = 256;  // threads per CTA of sep_tile_kernel
constexpr int SEP_SPLIT = 2;  // lanes sharing one (line, 8 outputs) tile (2: measured best)
template <typename TO>
__host__ __device__ constexpr int SEP_PAD() { return 16 / (int)sizeof(TO); }  // elements of line padding

template <typename TI, typename TO>
__global__ void __launch_bounds__(SEPT) sep_tile_kernel(const TI *__restrict__ in,
                                                        TO *__restrict__ out, int64_t batch,
                                                        int64_t cells, int L, int64_t S,
                                                        bool negate, int lpc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tpl = L / 8;
    TO *sq = reinterpret_cast<TO *>(smem_raw);          // [2L + 16]: sq[k] = (k - L - 7)^2
    // [lpc][LP]: lines padded by 16 bytes, so that the 16-byte reads of lanes on
    // consecutive lines (same source offset) fall into different banks -- a line
    // stride of L elements is a multiple of 128 bytes and made them all collide
    const int LP = L + SEP_PAD<TO>();
    TO *lines = sq + ((2 * L + 16 + 3) & ~3);
    const int64_t lines_per_pair = cells / L;
    const int64_t total_lines = batch * lines_per_pair;
    const int64_t line0 = (int64_t)blockIdx.x * lpc;
    // element offset of each of the CTA's lines (the 64-bit index arithmetic
    // once per line, not per element); -1 past the last line
    int64_t *lbase = reinterpret_cast<int64_t *>(lines + lpc * LP);
    for (int k = threadIdx.x; k < 2 * L + 16; k += blockDim.x) {
        const int d = k - L - 7;
        sq[k] = (TO)(d * d);
    }
    for (int li = threadIdx.x; li < lpc; li += blockDim.x) {
        const int64_t lid = line0 + li;
        int64_t off = -1;
        if (lid < total_lines) {
            const int64_t b = lid / lines_per_pair, r = lid - b * lines_per_pair;
            const int64_t low = r % S, high = r / S;
            off = b * cells + high * S * L + low;
        }
        lbase[li] = off;
    }
    __syncthreads();
    // load: consecutive threads -> consecutive lines (coalesced when S > 1);
    // contiguous axis: i fastest; strided axis: consecutive lines fastest
    for (int e = threadIdx.x; e < lpc * L; e += blockDim.x) {
        const int li = S == 1 ? e / L : e % lpc;  // 32-bit: e < lpc * L
        const int i = S == 1 ? e - li * L : e / lpc;
        const int64_t off = lbase[li];
        TO v = (TO)0;
        if (off >= 0) {
            v = (TO)in[off + (int64_t)i * S];
            if (negate) v = -v;
        }
        lines[li * LP + i] = v;
    }
    __syncthreads();
    // SEP_SPLIT consecutive lanes split the source range of a (line, 8
    // outputs) tile: more warps for latency hiding; the parts meet in a
    // shuffle min
    const int part = threadIdx.x % SEP_SPLIT, t = threadIdx.x / SEP_SPLIT;
    const int li = t % lpc, tl = t / lpc;
    const bool live = tl < tpl;
    const int64_t lid = line0 + li;
    const TO *line = lines + li * LP;
    const int j0 = 8 * (live ? tl : 0);
    TO best[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) best[r] = (TO)INFINITY;
    const int nch = L / 8;  // chunks of 8 sources, split evenly over the parts
    const int ib = live ? 8 * (part * nch / SEP_SPLIT) : L;
    const int ie = live ? 8 * ((part + 1) * nch / SEP_SPLIT) : L;
    for (int i0 = ib; i0 < ie; i0 += 8) {
        const TO *cp = sq + (i0 - j0 + L);  // squares of d = i0 - j0 - 7 + q, 16-byte aligned
        if constexpr (sizeof(TO) == 4) {
            float vs[8], Lq[16];
            const float4 a0 = reinterpret_cast<const float4 *>(line + i0)[0];
            const float4 a1 = reinterpret_cast<const float4 *>(line + i0)[1];
            vs[0] = a0.x; vs[1] = a0.y; vs[2] = a0.z; vs[3] = a0.w;
            vs[4] = a1.x; vs[5] = a1.y; vs[6] = a1.z; vs[7] = a1.w;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                const float4 t = reinterpret_cast<const float4 *>(cp)[c4];
                Lq[4 * c4] = t.x; Lq[4 * c4 + 1] = t.y; Lq[4 * c4 + 2] = t.z; Lq[4 * c4 + 3] = t.w;
            }
            minplus_row8<false, false>(Lq, vs, best);
        } else {
            TO vs[8], cst[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) vs[q] = line[i0 + q];
#pragma unroll
            for (int q = 0; q < 16; ++q) cst[q] = cp[q];
#pragma unroll
            for (int r8 = 0; r8 < 8; ++r8)
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    const TO cand = cst[s - r8 + 7] + vs[s];
                    best[r8] = cand < best[r8] ? cand : best[r8];
                }
        }
    }
#pragma unroll
    for (int sh = 1; sh < SEP_SPLIT; sh <<= 1)
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
            const TO o = __shfl_xor_sync(0xffffffffu, best[r8], sh);
            best[r8] = o < best[r8] ? o : best[r8];
        }
    if (!live || part || lid >= total_lines) return;
    TO *o = out + lbase[li];
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) o[(int64_t)(j0 + r8) * S] = best[r8];
}

template <typename TI, typename TO>
__global__ void sep_pass_kernel(const TI *__restrict__ in, TO *__restrict__ out, int64_t batch,
                                Grid g, int ax, bool negate) {
    extern __shared__ unsigned char smem_raw[];
    TO *line = reinterpret_cast<TO *>(smem_raw);
    const int64_t L = g.n[ax], S = g.stride[ax];
    const int64_t lines_per_pair = g.cells / L;
    const int64_t line_id = blockIdx.x;  // one CTA per line
    const int64_t b = line_id / lines_per_pair;
    const int64_t r = line_id - b * lines_per_pair;
    // decompose r into (low part below axis, high part above axis)
    const int64_t low = r % S, high = r / S;
    const int64_t base = b * g.cells + high * S * L + low;
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
        TO v = (TO)in[base + i * S];
        line[i] = negate ? -v : v;
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j < L; j += blockDim.x) {
        TO best = (TO)INFINITY;
        for (int64_t i = 0; i < L; ++i) {
            const int64_t d = i - j;
            const TO cand = (TO)(d * d) + line[i];
            best = cand < best ? cand : best;
        }
        out[base + j * S] = best;
    }
}

// ---------------------------------------------------------------------------
// brute force, fp64: thread per output, sources through shared memory
// ---------------------------------------------------------------------------
constexpr int BT = 256;     // threads per CTA
constexpr int BTILE = 1024; // sources per shared tile

__global__ void __launch_bounds__(BT) brute_f64_kernel(const double *__restrict__ v,
                                                       double *__restrict__ out, int64_t batch,
                                                       Grid g, double p,
                                                       const double *__restrict__ table) {
    __shared__ double sv[BTILE];
    __shared__ int sx[BTILE][GDT_MAX_DIM];
    const int64_t tiles_per_pair = (g.cells + BT - 1) / BT;
    const int64_t b = blockIdx.x / tiles_per_pair;
    const int64_t j = (blockIdx.x - b * tiles_per_pair) * BT + threadIdx.x;
    int xj[GDT_MAX_DIM];
    {
        int64_t rem = j < g.cells ? j : 0;
        for (int a = g.nd - 1; a >= 0; --a) {
            xj[a] = (int)(rem / g.stride[a]);
            rem -= xj[a] * g.stride[a];
        }
    }
    double best = INFINITY;
    for (int64_t i0 = 0; i0 < g.cells; i0 += BTILE) {
        const int cnt = (int)(g.cells - i0 < BTILE ? g.cells - i0 : BTILE);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt; t += BT) {
            sv[t] = v[b * g.cells + i0 + t];
            int64_t rem = i0 + t;
            for (int a = g.nd - 1; a >= 0; --a) {
                sx[t][a] = (int)(rem / g.stride[a]);
                rem -= sx[t][a] * g.stride[a];
            }
        }
        __syncthreads();
        for (int t = 0; t < cnt; ++t) {
            int64_t sq = 0;
            for (int a = 0; a < g.nd; ++a) {
                const int64_t d = sx[t][a] - xj[a];
                sq += d * d;
            }
            best = fmin(best, __dsub_rn(__ldg(table + sq), sv[t]));
        }
    }
    if (j < g.cells) out[b * g.cells + j] = best;
}

// ---------------------------------------------------------------------------
// brute force, fp32, Toeplitz-tiled (any d; rows along axis 0)
//   CTA: 128 threads x R=8 outputs = 1024 consecutive outputs along axis 0
//   (wrapping over rows when n0 < 1024); sources stream one axis-0 row
//   segment of S=8 at a time.
// ---------------------------------------------------------------------------
constexpr int FT = 128;   // threads
constexpr int FR = 8;     // outputs per thread (consecutive along axis 0)
constexpr int FS = 8;     // sources per inner step
constexpr int FROWS = 16; // source rows per shared stage


__device__ __forceinline__ unsigned long long pack2(float a, float b) {
    return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}

__device__ __forceinline__ void sub2(float c0, float c1, float v0, float v1, float &r0, float &r1) {
    unsigned long long rr;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(pack2(c0, c1)), "l"(pack2(v0, v1)));
    r0 = __uint_as_float((unsigned)(rr & 0xffffffffu));
    r1 = __uint_as_float((unsigned)(rr >> 32));
}

__device__ __forceinline__ float min3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__global__ void __launch_bounds__(FT) brute_f32_kernel(const float *__restrict__ v,
                                                       float *__restrict__ out, int64_t batch,
                                                       Grid g, double p,
                                                       const float *__restrict__ ftab) {
    // shared: FROWS source rows of n0 values
    extern __shared__ float sv[];
    const int64_t n0 = g.n[0];
    const int64_t outs_per_cta = FT * FR;
    const int64_t ctas_per_pair = (g.cells + outs_per_cta - 1) / outs_per_cta;
    const int64_t b = blockIdx.x / ctas_per_pair;
    const int64_t j0 = (blockIdx.x - b * ctas_per_pair) * outs_per_cta + (int64_t)threadIdx.x * FR;
    // outputs j0 .. j0+FR-1; require n0 % FR == 0 so they share one axis-0 row
    int xj[GDT_MAX_DIM];
    {
        int64_t rem = j0 < g.cells ? j0 : 0;
        for (int a = g.nd - 1; a >= 0; --a) {
            xj[a] = (int)(rem / g.stride[a]);
            rem -= xj[a] * g.stride[a];
        }
    }
    float best[FR];
#pragma unroll
    for (int r = 0; r < FR; ++r) best[r] = INFINITY;
    const int64_t rows = g.cells / n0;  // source rows (all higher coords)
    for (int64_t r0 = 0; r0 < rows; r0 += FROWS) {
        const int nr = (int)(rows - r0 < FROWS ? rows - r0 : FROWS);
        __syncthreads();
        for (int64_t t = threadIdx.x; t < nr * n0; t += FT) sv[t] = v[b * g.cells + r0 * n0 + t];
        __syncthreads();
        for (int rr = 0; rr < nr; ++rr) {
            // higher-axis squared distance of this source row
            int64_t rem = r0 + rr;
            int hsq = 0;
            for (int a = 1; a < g.nd; ++a) {
                const int64_t sa = g.n[a];
                const int xa = (int)(rem % sa);
                rem /= sa;
                const int d = xa - xj[a];
                hsq += d * d;
            }
            const float *row = sv + rr * n0;
            for (int s0 = 0; s0 < n0; s0 += FS) {
                // costs for dx = (s0 + s) - (xj0 + r), s in [0,FS), r in [0,FR)
                float cst[FR + FS - 1];
#pragma unroll
                for (int q = 0; q < FR + FS - 1; ++q) {
                    const int dx = s0 - xj[0] - (FR - 1) + q;
                    cst[q] = __ldg(ftab + hsq + dx * dx);
                }
                float vs[FS];
#pragma unroll
                for (int s = 0; s < FS; ++s) vs[s] = row[s0 + s];
#pragma unroll
                for (int r = 0; r < FR; ++r) {
#pragma unroll
                    for (int s = 0; s < FS; s += 2) {
                        float c0, c1;
                        sub2(cst[s - r + FR - 1], cst[s + 1 - r + FR - 1], vs[s], vs[s + 1], c0, c1);
                        best[r] = min3(best[r], c0, c1);
                    }
                }
            }
        }
    }
    if (j0 < g.cells) {
#pragma unroll
        for (int r = 0; r < FR; ++r) out[b * g.cells + j0 + r] = best[r];
    }
}

template <typename T>
__global__ void __launch_bounds__(1024) dot_mass_kernel(const T *__restrict__ x,
                                                        const double *__restrict__ m, int64_t n,
                                                        double *__restrict__ out) {
    __shared__ double sh[32];
    const int64_t b = blockIdx.x;
    const T *xb = x + b * n;
    const double *mb = m + b * n;
    // four independent partial sums per thread (loads in flight), fixed order
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t i = threadIdx.x;
    for (; i + 3 * 1024 < n; i += 4 * 1024) {
        a0 += (double)xb[i] * mb[i];
        a1 += (double)xb[i + 1024] * mb[i + 1024];
        a2 += (double)xb[i + 2048] * mb[i + 2048];
        a3 += (double)xb[i + 3072] * mb[i + 3072];
    }
    for (; i < n; i += 1024) a0 += (double)xb[i] * mb[i];
    double acc = (a0 + a1) + (a2 + a3);
    acc = block_sum<1024>(acc, sh);
    if (threadIdx.x == 0) out[b] = acc;
}

__global__ void f64_to_f32_kernel(const double *__restrict__ in, float *__restrict__ out, int64_t n,
                                  bool negate) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)(negate ? -in[i] : in[i]);
}

__global__ void table_to_f32_kernel(const double *__restrict__ in, float *__restrict__ out,
                                    int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

// ---------------------------------------------------------------------------
// point-cloud c-transform (fp64), CostSpec semantics
// ---------------------------------------------------------------------------
__global__ void points_ct_kernel(const double *__restrict__ xo, const double *__restrict__ xi,
                                 int64_t no, int64_t ni, int nd, double p,
                                 const double *__restrict__ v, double *__restrict__ out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= no) return;
    double best = INFINITY;
    for (int64_t i = 0; i < ni; ++i) {
        double sq = 0.0;
        for (int a = 0; a < nd; ++a) {
            const double d = __dsub_rn(xi[i * nd + a], xo[j * nd + a]);
            sq = __dadd_rn(sq, __dmul_rn(d, d));
        }
        double c = p == 2.0 ? sq : (p == 1.0 ? __dsqrt_rn(sq) : pow(sq, p / 2.0));
        best = fmin(best, __dsub_rn(c, v[i]));
    }
    out[j] = best;
}

}  // namespace gdt

namespace gdt {
int ct_pruned_f32(const float *v, float *out, float *tmax, int64_t batch, const Grid &g, double p,
                  const float *ftab, cudaStream_t st);
int ct_pruned_f64(const double *v, double *out, double *tmax, int64_t batch, const Grid &g,
                  double p, const double *tab, cudaStream_t st);
int64_t ct_pruned_tiles(const Grid &g);
}  // namespace gdt

using namespace gdt;

extern "C" int64_t gdt_ctransform_scratch_bytes(int64_t batch, int ndim, const int64_t *dims,
                                                double p, int dtype) {
    Grid g;
    if (!make_grid(g, ndim, dims)) return -1;
    const int64_t el = dtype == 0 ? 8 : 4;
    int64_t need_sq = 0;
    for (int a = 0; a < ndim; ++a) need_sq += (dims[a] - 1) * (dims[a] - 1);
    // ping-pong buffer (+ fp32 input copy) + fp32 cost table + pruning tile maxima
    return batch * g.cells * el * 2 + (need_sq + 1) * 4 + batch * ct_pruned_tiles(g) * 8 + 1024;
}

extern "C" int gdt_ctransform_grid(const void *v, void *out, int64_t batch, int ndim,
                                   const int64_t *dims, double p, int dtype, int in_dtype,
                                   const double *cost_table, int64_t max_sq, const double *mass,
                                   double *dot_out, void *scratch, int64_t scratch_bytes,
                                   void *stream) {
    Grid g;
    GDT_CHECK_ARG(make_grid(g, ndim, dims) && p >= 1.0 && batch >= 0,
                  "gdt_ctransform_grid: bad grid or p");
    GDT_CHECK_ARG((dtype == 0 || dtype == 1) && (in_dtype == 0 || in_dtype == 1),
                  "gdt_ctransform_grid: dtype must be 0 (fp64) or 1 (fp32)");
    GDT_CHECK_ARG(in_dtype == dtype || (in_dtype == 0 && dtype == 1),
                  "gdt_ctransform_grid: fp32 input needs fp32 output");
    int64_t need_sq = 0;
    for (int a = 0; a < ndim; ++a) need_sq += (dims[a] - 1) * (dims[a] - 1);
    GDT_CHECK_ARG(p == 2.0 || (cost_table != nullptr && max_sq >= need_sq),
                  "gdt_ctransform_grid: cost_table required for p != 2");
    GDT_CHECK_ARG(scratch_bytes >= gdt_ctransform_scratch_bytes(batch, ndim, dims, p, dtype),
                  "gdt_ctransform_grid: scratch too small");
    if (batch == 0) return GDT_OK;
    cudaStream_t st = as_stream(stream);
    const int64_t total = batch * g.cells;
    char *scr = (char *)scratch;
    if (p == 2.0) {
        // d passes; the first negates its input; ping-pong out <-> scratch so
        // that the last pass lands in `out`
        const int64_t el = dtype == 0 ? 8 : 4;
        void *bufs[2] = {out, scr};
        int dst = (ndim % 2 == 1) ? 0 : 1;  // pass 0 target so that pass d-1 -> out
        const void *src = v;
        int src_dtype = in_dtype;
        for (int ax = 0; ax < ndim; ++ax) {
            const int64_t L = g.n[ax];
            void *o = bufs[dst];
            if (L % 8 == 0 && L / 8 <= SEPT / SEP_SPLIT) {
                // lines per CTA: fill the CTA, but keep >= 2 CTAs per SM
                const int tpl = (int)(L / 8);
                int dev = 0, nsm = 148;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
                const int64_t lines = total / L;
                int lpc = SEPT / (SEP_SPLIT * tpl);  // SEP_SPLIT threads per (line, 8 outputs)
                while (lpc > 1 && (lines + lpc - 1) / lpc < 2 * nsm) lpc >>= 1;
                const int thr = ((SEP_SPLIT * lpc * tpl + 31) / 32) * 32;
                const unsigned ctas = (unsigned)((lines + lpc - 1) / lpc);
                const size_t sh = el * (((2 * L + 16 + 3) & ~3) + (size_t)lpc * (L + 16 / el)) +
                                  sizeof(int64_t) * lpc;  // padded lines + line offsets
                if (dtype == 0)
                    sep_tile_kernel<double, double><<<ctas, thr, sh, st>>>(
                        (const double *)src, (double *)o, batch, g.cells, (int)L, g.stride[ax], ax == 0, lpc);
                else if (src_dtype == 0)
                    sep_tile_kernel<double, float><<<ctas, thr, sh, st>>>(
                        (const double *)src, (float *)o, batch, g.cells, (int)L, g.stride[ax], ax == 0, lpc);
                else
                    sep_tile_kernel<float, float><<<ctas, thr, sh, st>>>(
                        (const float *)src, (float *)o, batch, g.cells, (int)L, g.stride[ax], ax == 0, lpc);
                src = o;
                src_dtype = dtype;
                dst ^= 1;
                continue;
            }
            const unsigned ctas = (unsigned)(total / L);
            const int thr = L >= 256 ? 256 : (int)((L + 31) / 32 * 32);
            const size_t sh = L * el;
            if (dtype == 0)
                sep_pass_kernel<double, double><<<ctas, thr, sh, st>>>(
                    (const double *)src, (double *)o, batch, g, ax, ax == 0);
            else if (src_dtype == 0)
                sep_pass_kernel<double, float><<<ctas, thr, sh, st>>>(
                    (const double *)src, (float *)o, batch, g, ax, ax == 0);
            else
                sep_pass_kernel<float, float><<<ctas, thr, sh, st>>>(
                    (const float *)src, (float *)o, batch, g, ax, ax == 0);
            src = o;
            src_dtype = dtype;
            dst ^= 1;
            (void)el;
        }
    } else if (dtype == 0) {
        double *tmax = (double *)(scr + total * 8 * 2 + ((need_sq + 1) * 4 + 255) / 256 * 256);
        if (ct_pruned_f64((const double *)v, (double *)out, tmax, batch, g, p, cost_table, st) !=
            GDT_OK) {
            const int64_t tiles = (g.cells + BT - 1) / BT;
            brute_f64_kernel<<<(unsigned)(batch * tiles), BT, 0, st>>>(
                (const double *)v, (double *)out, batch, g, p, cost_table);
        }
    } else {
        GDT_CHECK_ARG(g.n[0] % FR == 0, "gdt_ctransform_grid: fp32 brute needs dims[0] % 8 == 0");
        float *vin = (float *)scr;
        float *ftab = (float *)(scr + total * 4 * 2);
        const float *vsrc = (const float *)v;
        if (in_dtype == 0) {
            f64_to_f32_kernel<<<grid_size(total, 256) > 2048 ? 2048 : grid_size(total, 256), 256, 0,
                                st>>>((const double *)v, vin, total, false);
            vsrc = vin;
        }
        table_to_f32_kernel<<<grid_size(need_sq + 1, 256), 256, 0, st>>>(cost_table, ftab,
                                                                             need_sq + 1);
        float *tmax = (float *)(scr + total * 4 * 2 + ((need_sq + 1) * 4 + 255) / 256 * 256);
        if (ct_pruned_f32(vsrc, (float *)out, tmax, batch, g, p, ftab, st) == GDT_OK) {
            vsrc = nullptr;  // done
        }
        const int64_t per = FT * FR;
        const int64_t ctas = batch * ((g.cells + per - 1) / per);
        const size_t sh = (size_t)FROWS * g.n[0] * 4;
        if (sh > 48 * 1024)
            cudaFuncSetAttribute(brute_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sh);
        if (vsrc != nullptr)
            brute_f32_kernel<<<(unsigned)ctas, FT, sh, st>>>(vsrc, (float *)out, batch, g, p, ftab);
    }
    if (mass != nullptr && dot_out != nullptr) {
        if (dtype == 0)
            dot_mass_kernel<double><<<(unsigned)batch, 1024, 0, st>>>((const double *)out, mass,
                                                                    g.cells, dot_out);
        else
            dot_mass_kernel<float><<<(unsigned)batch, 1024, 0, st>>>((const float *)out, mass,
                                                                   g.cells, dot_out);
    }
    return cuda_status("gdt_ctransform_grid");
}

extern "C" int gdt_ctransform_points(const double *xs, const double *xt, int64_t ns, int64_t nt,
                                     int ndim, double p, const double *v, int direction,
                                     double *out, void *stream) {
    GDT_CHECK_ARG(ns >= 1 && nt >= 1 && ndim >= 1 && p >= 1.0, "gdt_ctransform_points: bad args");
    GDT_CHECK_ARG(direction == 0 || direction == 1, "gdt_ctransform_points: bad direction");
    cudaStream_t st = as_stream(stream);
    if (direction == 0)  // out_j over targets, min over sources
        points_ct_kernel<<<grid_size(nt, 128), 128, 0, st>>>(xt, xs, nt, ns, ndim, p, v, out);
    else
        points_ct_kernel<<<grid_size(ns, 128), 128, 0, st>>>(xs, xt, ns, nt, ndim, p, v, out);
    return cuda_status("gdt_ctransform_points");
}
