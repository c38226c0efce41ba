// K4-K6: primal upscaling -- block-sparse IPF, pricing and TV inner sums.
//
// Reference: primal_upscaling_upper_bound (quantized.py:288-380) builds the
// fine coupling pi_hat_{(k,t),(l,s)} = m_kl * W[t,s] (upscale_coupling,
// quantized.py:119-159), restricts it to the supports into a canonical CSR
// (quantized.py:322-333) and runs ipf_fit (sinkhorn.py:101-142), whose
// products are scipy CSR/CSC mat-vecs: every row sum runs sequentially over
// ascending fine column, every column sum over ascending fine row.
//
// Here the fine coupling is never materialised.  For row block k the sorted
// columns of a CSR row are the cells of the arcs' target blocks in ascending
// fine flat index; `walk` enumerates exactly that order from the sorted arc
// list (lexicographic over (l_{d-1}, s_{d-1}, ..., l_0, s_0)).  With the
// uniform kernel every row of block k has the same term sequence, so one
// sequential fp64 sum per coarse block replaces kappa^d row sums and the
// result is bit-identical to scipy's.  Non-uniform kernels get one sum per
// fine row (W[t,s] depends on the row offset t).
//
// ipf_kernel: one CTA per pair stays resident for all sweeps; a sweep is two
// barrier-separated phases plus one block reduction:
//   C: per column unit: kta = sum coef * a_i (ascending rows); for its cells
//      b_j = nu_j / kta, |nu_j - b_j kta| into the gap, range(b), zero check;
//   R: per row unit: kb = sum coef * b_j (ascending columns); for its cells
//      |a_i kb - mu_i| with the current a, range(a), next a = mu_i / kb and
//      the zero-row check of the next sweep;
// applying the reference's checks in its order (sinkhorn.py:125-141).
// Then, grid-parallel and deterministic (no atomics):
//   moments_tv_kernel: per block, weighted-TV partials and the 0th/1st/2nd
//     moments of a and b about the block centre;
//   price_kernel: per arc, sum_{t,s} ((a_t m W_ts) b_s) C_ts -- in closed form
//     from the moments when p == 2 with the uniform kernel (the cost is a
//     quadratic), by direct summation with tabulated costs otherwise;
//   finish_kernel: fixed-order reduction of the per-CTA partials.
#include <cstdlib>

#include "common.cuh"

namespace gdt {

constexpr int PT = 512;  // threads of the per-pair IPF CTA (128 registers each)
constexpr int CL_SKEW = 2;  // doubles of shared-memory skew per unit (ipf_cluster_kernel products)

struct G32 {  // int32 grid description (cells < 2^31)
    int nd;
    int n[GDT_MAX_DIM];
    int stride[GDT_MAX_DIM];
    int cells;
};

inline G32 to32(const Grid &g) {
    G32 o;
    o.nd = g.nd;
    for (int a = 0; a < GDT_MAX_DIM; ++a) {
        o.n[a] = (int)g.n[a];
        o.stride[a] = (int)g.stride[a];
    }
    o.cells = (int)g.cells;
    return o;
}

__device__ __forceinline__ int coord_of(int id, const G32 &c, int a) {
    return (id / c.stride[a]) % c.n[a];
}

// fine flat id of the origin cell of block k
__device__ __forceinline__ int block_origin(int k, const G32 &c, const G32 &f, int kappa) {
    int off = 0;
    for (int a = c.nd - 1; a >= 0; --a) {
        const int ka = k / c.stride[a];
        k -= ka * c.stride[a];
        off += ka * kappa * f.stride[a];
    }
    return off;
}

// visit the kappa^d cells of a block in ascending fine order: fn(offset_index, cell)
template <class F>
__device__ __forceinline__ void for_block_cells(int origin, const G32 &f, int kappa, F &&fn) {
    const int K1 = f.nd > 1 ? kappa : 1, K2 = f.nd > 2 ? kappa : 1, K3 = f.nd > 3 ? kappa : 1;
    int t = 0;
    for (int o3 = 0; o3 < K3; ++o3)
        for (int o2 = 0; o2 < K2; ++o2)
            for (int o1 = 0; o1 < K1; ++o1) {
                const int row = origin + o3 * f.stride[3] + o2 * f.stride[2] + o1 * f.stride[1];
                for (int o0 = 0; o0 < kappa; ++o0, ++t) fn(t, row + o0);
            }
}

// Visit the cells of the union of coarse blocks of arcs [lo, hi) (sorted by
// coarse id) in ascending fine flat order, as runs of kappa consecutive cells
// along axis 0: fn(q, cell, s) with q the arc index, cell the fine flat id of
// the run's first cell and s its within-block offset (Fortran-flattened).
// pc[q] packs the arc's coarse coordinates, 16 bits per axis (axis 0 lowest).
__device__ __forceinline__ int pc_coord(int64_t w, int a) { return (int)((w >> (16 * a)) & 0xffff); }

template <int LEVEL, class F>
__device__ __forceinline__ void walk(const int64_t *pc, int lo, int hi, const G32 &f, int kappa,
                                     int fbase, int sbase, int kpow, F &fn) {
    if constexpr (LEVEL == 0) {
        // one run of kappa consecutive cells per arc: fn(q, first_cell, first_s)
        for (int q = lo; q < hi; ++q) fn(q, fbase + pc_coord(pc[q], 0) * kappa, sbase);
    } else {
        int r = lo;
        while (r < hi) {
            const int cr = pc_coord(pc[r], LEVEL);
            int e = r + 1;
            while (e < hi && pc_coord(pc[e], LEVEL) == cr) ++e;
            for (int sa = 0; sa < kappa; ++sa)
                walk<LEVEL - 1>(pc, r, e, f, kappa, fbase + (cr * kappa + sa) * f.stride[LEVEL],
                                sbase + sa * kpow, kpow / kappa, fn);
            r = e;
        }
    }
}

template <class F>
__device__ __forceinline__ void walk_blocks(const int64_t *pc, int cnt, const G32 &c,
                                            const G32 &f, int kappa, F &fn) {
    const int kpow = (int)ipow(kappa, c.nd - 1);
    switch (c.nd) {
        case 1: walk<0>(pc, 0, cnt, f, kappa, 0, 0, kpow, fn); break;
        case 2: walk<1>(pc, 0, cnt, f, kappa, 0, 0, kpow, fn); break;
        case 3: walk<2>(pc, 0, cnt, f, kappa, 0, 0, kpow, fn); break;
        default: walk<3>(pc, 0, cnt, f, kappa, 0, 0, kpow, fn); break;
    }
}

// packed coarse coordinates of every arc endpoint (row lists: targets, column
// lists: sources), built once per launch
__global__ void pack_coords_kernel(const int32_t *__restrict__ ids, const int64_t *__restrict__ arc_off,
                                   int64_t per_pair, int64_t batch, G32 c,
                                   int64_t *__restrict__ pc) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < batch * per_pair;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per_pair, q = t - b * per_pair;
        if (q >= arc_off[b + 1] - arc_off[b]) continue;
        const int64_t i = arc_off[b] + q;
        int id = ids[i];
        int64_t w = 0;
        for (int a = c.nd - 1; a >= 0; --a) {
            const int x = id / c.stride[a];
            id -= x * c.stride[a];
            w |= (int64_t)x << (16 * a);
        }
        pc[i] = w;
    }
}

struct PairPtrs {
    const double *mu, *nu;
    const int32_t *rptr, *rcol, *cptr, *crow;
    const int64_t *rpc, *cpc;
    const double *rmass, *cmass;
    double *aA, *aB, *b, *kb, *kta;
    // uniform kernel: the walk of every unit precomputed once per launch as
    // runs (first cell, coefficient mass * W), arc q owning runs
    // [q * K1, (q + 1) * K1), K1 = kappa^(d-1) (run_list_par_kernel)
    const int32_t *rrc, *crc;
    const double *rrf, *crf;
    int pf;  // the gathered vector is in global memory: prefetch runs into L1
};

constexpr int PF_RUNS = 8;  // runs prefetched ahead of the exact-order adds

#ifdef GDT_IPF_TRACE
// debug builds: SM clock at the phase boundaries of sweep 10 of pair 0
__device__ long long g_ex_trace[16];
#define EX_TRACE(slot_)                                                   \
    do {                                                                  \
        if (blockIdx.x == 0 && threadIdx.x == 0 && it == 10) g_ex_trace[(slot_)] = clock64(); \
    } while (0)
#else
#define EX_TRACE(slot_) \
    do {                \
    } while (0)
#endif

__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Exact-order run sum of one unit from its precomputed run list: runs are
// consumed in order, the next run's loads issued before the current run's
// adds (they do not depend on acc), every term rounded as accumulate_run does.
template <int KAP>
__device__ __forceinline__ double run_list_sum(const int32_t *cells, const double *coefs, int nr,
                                               const double *x, int pf) {
    double acc = 0.0;
    if (nr <= 0) return acc;
    // global-memory vector: the unit is a chain of dependent adds whose loads
    // are known in advance, so the next PF_RUNS runs are pulled into L1 first
    // (their latency then overlaps the adds; no register cost)
    if (pf)
        for (int r = 0; r < nr && r < PF_RUNS; ++r) prefetch_l1(x + cells[r]);
    double xc[KAP], cc = coefs[0];
    {
        const double *p0 = x + cells[0];
#pragma unroll
        for (int i = 0; i < KAP; ++i) xc[i] = p0[i];
    }
    for (int r = 0; r < nr; ++r) {
        double xn[KAP], cn = 0.0;
        if (pf && r + PF_RUNS < nr) prefetch_l1(x + cells[r + PF_RUNS]);
        if (r + 1 < nr) {
            const double *pn = x + cells[r + 1];
            cn = coefs[r + 1];
#pragma unroll
            for (int i = 0; i < KAP; ++i) xn[i] = pn[i];
        }
#pragma unroll
        for (int i = 0; i < KAP; ++i) acc = __dadd_rn(acc, __dmul_rn(cc, xc[i]));
#pragma unroll
        for (int i = 0; i < KAP; ++i) xc[i] = xn[i];
        cc = cn;
    }
    return acc;
}

__device__ __forceinline__ double run_list_sum_any(const int32_t *cells, const double *coefs,
                                                   int nr, const double *x, int kappa, int pf) {
    switch (kappa) {
        case 2: return run_list_sum<2>(cells, coefs, nr, x, pf);
        case 4: return run_list_sum<4>(cells, coefs, nr, x, pf);
        default: {
            double acc = 0.0;
            for (int r = 0; r < nr; ++r) {
                const double cf = coefs[r], *p = x + cells[r];
                for (int i = 0; i < kappa; ++i) acc = __dadd_rn(acc, __dmul_rn(cf, p[i]));
            }
            return acc;
        }
    }
}

// Uniform kernel, kappa <= 8: the unit sums in two phases.  (1) Every
// product coef * x of every run of every unit, in parallel over the runs,
// written in chain order into a contiguous buffer; (2) one sequential fp64
// sum per unit over its contiguous products.  The products and the order of
// the adds are those of run_list_sum (= scipy's CSR/CSC matvec order), so the
// sums are bit-identical -- but the dependent chain of a long unit now only
// waits for adds, not for a gather per run.
template <int KAP>
__device__ __forceinline__ void run_products(const int32_t *__restrict__ cells,
                                             const double *__restrict__ coefs, int nruns,
                                             const double *__restrict__ x,
                                             double *__restrict__ prod, int kappa) {
    if constexpr (KAP >= 2 && KAP <= 4) {
        // RU runs per thread at a time: run descriptors, then the gathers, then
        // the products (the loads of a group are all in flight together)
        constexpr int RU = 4;
        for (int r0 = threadIdx.x; r0 < nruns; r0 += PT * RU) {
            int cl[RU];
            double cf[RU], xv[RU][KAP];
#pragma unroll
            for (int q = 0; q < RU; ++q) {
                const int r = r0 + q * PT;
                cl[q] = r < nruns ? cells[r] : 0;
                cf[q] = r < nruns ? coefs[r] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < RU; ++q)
#pragma unroll
                for (int i = 0; i < KAP; ++i) xv[q][i] = r0 + q * PT < nruns ? x[cl[q] + i] : 0.0;
#pragma unroll
            for (int q = 0; q < RU; ++q) {
                const int r = r0 + q * PT;
                if (r >= nruns) break;
                double *pp = prod + (int64_t)r * KAP;
#pragma unroll
                for (int i = 0; i < KAP; i += 2)
                    *reinterpret_cast<double2 *>(pp + i) =
                        make_double2(__dmul_rn(cf[q], xv[q][i]), __dmul_rn(cf[q], xv[q][i + 1]));
            }
        }
    } else {
        for (int r = threadIdx.x; r < nruns; r += PT) {
            const double cf = coefs[r];
            const double *xp = x + cells[r];
            if constexpr (KAP >= 2) {
                double *pp = prod + (int64_t)r * KAP;
#pragma unroll
                for (int i = 0; i < KAP; i += 2)
                    *reinterpret_cast<double2 *>(pp + i) =
                        make_double2(__dmul_rn(cf, xp[i]), __dmul_rn(cf, xp[i + 1]));
            } else {
                double *pp = prod + (int64_t)r * kappa;
                for (int i = 0; i < kappa; ++i) pp[i] = __dmul_rn(cf, xp[i]);
            }
        }
    }
}

// acc = (((0 + p0) + p1) + ...) over `len` contiguous products in shared
// memory (16-byte aligned when `vec`).  Software-pipelined: the next 8
// products are loaded while the current 8 are added, so the chain waits only
// on the adds.
__device__ __forceinline__ double chain_sum(const double *__restrict__ p, int len, bool vec) {
    double acc = 0.0;
    int j = 0;
    if (vec && len >= 8) {
        const double2 *q = reinterpret_cast<const double2 *>(p);
        double2 c0 = q[0], c1 = q[1], c2 = q[2], c3 = q[3];
        for (; j + 16 <= len; j += 8) {
            const double2 *qn = reinterpret_cast<const double2 *>(p + j + 8);
            const double2 n0 = qn[0], n1 = qn[1], n2 = qn[2], n3 = qn[3];
            acc = __dadd_rn(acc, c0.x);
            acc = __dadd_rn(acc, c0.y);
            acc = __dadd_rn(acc, c1.x);
            acc = __dadd_rn(acc, c1.y);
            acc = __dadd_rn(acc, c2.x);
            acc = __dadd_rn(acc, c2.y);
            acc = __dadd_rn(acc, c3.x);
            acc = __dadd_rn(acc, c3.y);
            c0 = n0;
            c1 = n1;
            c2 = n2;
            c3 = n3;
        }
        acc = __dadd_rn(acc, c0.x);
        acc = __dadd_rn(acc, c0.y);
        acc = __dadd_rn(acc, c1.x);
        acc = __dadd_rn(acc, c1.y);
        acc = __dadd_rn(acc, c2.x);
        acc = __dadd_rn(acc, c2.y);
        acc = __dadd_rn(acc, c3.x);
        acc = __dadd_rn(acc, c3.y);
        j += 8;
    }
    for (; j < len; ++j) acc = __dadd_rn(acc, p[j]);
    return acc;
}

// out[u] = the exact-order sum of unit u for every unit of the pair.  The
// products of consecutive units are staged batch by batch (at most `cap`
// doubles of shared memory per batch); a unit whose products alone exceed
// `cap` is summed straight from its run list.
__device__ __noinline__ void unit_sums(const int32_t *cells, const double *coefs,
                                       const int32_t *ptr, int U, int K1, int kappa,
                                       const double *x, double *prod, double *out, int cap,
                                       int pf) {
    const int per = K1 * kappa;  // products per arc
    const bool vec = (per & 1) == 0;
    int u0 = 0;
    while (u0 < U) {
        // the batch [u0, u1): as many whole units as fit (every thread computes
        // the same boundary); an oversized unit forms a batch of its own
        const int a0 = ptr[u0];
        int lo = u0 + 1, hi = U;  // largest u1 in [u0 + 1, U] whose products fit
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int64_t)(ptr[mid] - a0) * per <= cap) lo = mid;
            else hi = mid - 1;
        }
        const int u1 = lo;
        const bool staged = (int64_t)(ptr[u1] - a0) * per <= cap;
        if (staged) {
            const int nruns = (ptr[u1] - a0) * K1;
            const int32_t *bc = cells + (int64_t)a0 * K1;
            const double *bf = coefs + (int64_t)a0 * K1;
            switch (kappa) {
                case 2: run_products<2>(bc, bf, nruns, x, prod, kappa); break;
                case 4: run_products<4>(bc, bf, nruns, x, prod, kappa); break;
                case 8: run_products<8>(bc, bf, nruns, x, prod, kappa); break;
                default: run_products<0>(bc, bf, nruns, x, prod, kappa); break;
            }
            __syncthreads();
            for (int u = u0 + (int)threadIdx.x; u < u1; u += PT) {
                const int64_t lo = (int64_t)(ptr[u] - a0) * per, hi = (int64_t)(ptr[u + 1] - a0) * per;
                out[u] = chain_sum(prod + lo, (int)(hi - lo), vec);
            }
            __syncthreads();  // before the next batch overwrites the products
        } else if (threadIdx.x == 0) {
            const int lo = ptr[u0] * K1, hi = ptr[u0 + 1] * K1;
            out[u0] = run_list_sum_any(cells + lo, coefs + lo, hi - lo, x, kappa, pf);
        }
        u0 = u1;
    }
}

struct Red {  // per-sweep reduction slots
    double gap, amin, amax, bmin, bmax;
    int zrow, zcol, nonfinite;
};

__device__ __forceinline__ Red red_init() {
    return Red{0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0, 0, 0};
}

__device__ __forceinline__ void range_acc(double v, double &lo, double &hi, int &nonfinite) {
    if (v > 0.0) {
        lo = fmin(lo, v);
        hi = fmax(hi, v);
        if (!isfinite(v)) nonfinite = 1;
    } else if (isnan(v)) {
        nonfinite = 1;
    }
}

__device__ void block_reduce_red(Red &r, double *sh) {
    // warp butterflies, then warp 0 folds the per-warp records the same way
    // and publishes the result (sh holds (PT / 32 + 1) * 6 doubles)
    auto warp_fold = [](Red &x) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            x.gap += __shfl_xor_sync(0xffffffffu, x.gap, o);
            x.amin = fmin(x.amin, __shfl_xor_sync(0xffffffffu, x.amin, o));
            x.bmin = fmin(x.bmin, __shfl_xor_sync(0xffffffffu, x.bmin, o));
            x.amax = fmax(x.amax, __shfl_xor_sync(0xffffffffu, x.amax, o));
            x.bmax = fmax(x.bmax, __shfl_xor_sync(0xffffffffu, x.bmax, o));
            x.zrow |= __shfl_xor_sync(0xffffffffu, x.zrow, o);
            x.zcol |= __shfl_xor_sync(0xffffffffu, x.zcol, o);
            x.nonfinite |= __shfl_xor_sync(0xffffffffu, x.nonfinite, o);
        }
    };
    warp_fold(r);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int NW = PT / 32;
    static_assert(NW <= 32, "one warp folds the per-warp records");
    __syncthreads();
    if (lane == 0) {
        sh[w * 6 + 0] = r.gap;
        sh[w * 6 + 1] = r.amin;
        sh[w * 6 + 2] = r.amax;
        sh[w * 6 + 3] = r.bmin;
        sh[w * 6 + 4] = r.bmax;
        sh[w * 6 + 5] = (double)(r.zrow | (r.zcol << 1) | (r.nonfinite << 2));
    }
    __syncthreads();
    if (w == 0) {
        Red o = red_init();
        if (lane < NW) {
            o.gap = sh[lane * 6 + 0];
            o.amin = sh[lane * 6 + 1];
            o.amax = sh[lane * 6 + 2];
            o.bmin = sh[lane * 6 + 3];
            o.bmax = sh[lane * 6 + 4];
            const int fl = (int)sh[lane * 6 + 5];
            o.zrow = fl & 1;
            o.zcol = (fl >> 1) & 1;
            o.nonfinite = (fl >> 2) & 1;
        }
        warp_fold(o);
        if (lane == 0) {
            double *res = sh + NW * 6;
            res[0] = o.gap;
            res[1] = o.amin;
            res[2] = o.amax;
            res[3] = o.bmin;
            res[4] = o.bmax;
            res[5] = (double)(o.zrow | (o.zcol << 1) | (o.nonfinite << 2));
        }
    }
    __syncthreads();
    const double *res = sh + NW * 6;
    r.gap = res[0];
    r.amin = res[1];
    r.amax = res[2];
    r.bmin = res[3];
    r.bmax = res[4];
    const int fl = (int)res[5];
    r.zrow = fl & 1;
    r.zcol = (fl >> 1) & 1;
    r.nonfinite = (fl >> 2) & 1;
    __syncthreads();
}

// Correctly rounded num / den for many numerators sharing one denominator:
// y = RN(1/den) once, then q = RN(num*y), r = num - den*q (exact with FMA),
// q' = RN(q + r*y) -- Markstein's theorem gives q' = RN(num/den) whenever no
// intermediate leaves the normal range, which the guard checks (otherwise the
// IEEE division routine runs).  Bit-identical to numpy's `mu / kb`.
__device__ __forceinline__ double div_shared(double num, double den, double y) {
    const double an = fabs(num), ad = fabs(den);
    if (an > 0x1p-900 && an < 0x1p900 && ad > 0x1p-900 && ad < 0x1p900) {
        const double q = __dmul_rn(num, y);
        const double r = __fma_rn(-q, den, num);
        return __fma_rn(r, y, q);
    }
    return __ddiv_rn(num, den);
}

// acc += (mass * w_i) * x_i sequentially over a run of `len` cells; the loads
// are issued first (they do not depend on acc), then the exact-order adds.
// Non-uniform kernels read w_i = wrow[i * wstride].
template <bool UNIFORM>
__device__ __forceinline__ void accumulate_run(double &acc, double mass, double Wu,
                                               const double *wrow, int wstride,
                                               const double *x, int len) {
    if (UNIFORM && (len & 1) == 0) {
        // 16-byte loads (kappa even), issued ahead of the exact-order adds
        const double coef = __dmul_rn(mass, Wu);
        for (int o = 0; o < len; o += 4) {
            const double2 x0 = reinterpret_cast<const double2 *>(x + o)[0];
            const double2 x1 = o + 2 < len ? reinterpret_cast<const double2 *>(x + o)[1]
                                           : make_double2(0.0, 0.0);
            acc = __dadd_rn(acc, __dmul_rn(coef, x0.x));
            acc = __dadd_rn(acc, __dmul_rn(coef, x0.y));
            if (o + 2 < len) {
                acc = __dadd_rn(acc, __dmul_rn(coef, x1.x));
                acc = __dadd_rn(acc, __dmul_rn(coef, x1.y));
            }
        }
        return;
    }
    for (int o = 0; o < len; o += 4) {
        double xv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) xv[i] = o + i < len ? x[o + i] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (o + i >= len) break;
            const double coef = __dmul_rn(mass, UNIFORM ? Wu : wrow[(o + i) * wstride]);
            acc = __dadd_rn(acc, __dmul_rn(coef, xv[i]));
        }
    }
}

// Phase R for one row unit (block k, or fine row (k, t) for non-uniform W).
template <bool UNIFORM>
__device__ __forceinline__ void row_unit(int u, const PairPtrs &P, const G32 &c, const G32 &f,
                                         int kappa, int m, const double *W, double Wu, bool init,
                                         const double *a_cur, double *a_next, Red &r,
                                         const double *bsrc) {
    const int k = UNIFORM ? u : u / m;
    const int t = UNIFORM ? 0 : u - k * m;
    const int lo = P.rptr[k], hi = P.rptr[k + 1];
    if (UNIFORM && kappa <= 8) {  // cells handled by cell_pass_row (all threads, all cells)
        const int K1 = m / kappa;
        P.kb[u] = run_list_sum_any(P.rrc + lo * K1, P.rrf + lo * K1, (hi - lo) * K1, bsrc, kappa,
                                   P.pf);
        return;
    }
    const int64_t *ids = P.rpc + lo;
    const double *ms = P.rmass + lo;
    double acc = 0.0;
    auto fn = [&](int q, int cell, int s) {
        accumulate_run<UNIFORM>(acc, ms[q], Wu, W + t * m + s, 1, bsrc + cell, kappa);
    };
    walk_blocks(ids, hi - lo, c, f, kappa, fn);
    P.kb[u] = acc;
    if (UNIFORM) return;
    const double rcp = acc > 0.0 ? __drcp_rn(acc) : 0.0;
    const int origin = block_origin(k, c, f, kappa);
    for_block_cells(origin, f, kappa, [&](int tt, int i) {
        if (!UNIFORM && tt != t) return;
        const double mui = P.mu[i];
        if (!init) {
            const double ai = a_cur[i];
            range_acc(ai, r.amin, r.amax, r.nonfinite);
            if (mui > 0.0) r.gap += fabs(__dsub_rn(__dmul_rn(ai, acc), mui));
        }
        double an = 0.0;
        if (mui > 0.0) {
            if (acc <= 0.0) r.zrow = 1;
            else an = div_shared(mui, acc, rcp);
        }
        a_next[i] = an;
    });
}

template <bool UNIFORM>
__device__ __forceinline__ void col_unit(int u, const PairPtrs &P, const G32 &c, const G32 &f,
                                         int kappa, int m, const double *W, double Wu,
                                         const double *a_cur, Red &r, const double *asrc) {
    const int l = UNIFORM ? u : u / m;
    const int s = UNIFORM ? 0 : u - l * m;
    const int lo = P.cptr[l], hi = P.cptr[l + 1];
    if (UNIFORM && kappa <= 8) {  // cells handled by cell_pass_col
        const int K1 = m / kappa;
        P.kta[u] = run_list_sum_any(P.crc + lo * K1, P.crf + lo * K1, (hi - lo) * K1, asrc, kappa,
                                    P.pf);
        return;
    }
    const int64_t *ids = P.cpc + lo;
    const double *ms = P.cmass + lo;
    double acc = 0.0;
    auto fn = [&](int q, int cell, int t) {
        accumulate_run<UNIFORM>(acc, ms[q], Wu, W + t * m + s, m, asrc + cell, kappa);
    };
    walk_blocks(ids, hi - lo, c, f, kappa, fn);
    P.kta[u] = acc;
    if (UNIFORM) return;
    const double rcp = acc > 0.0 ? __drcp_rn(acc) : 0.0;
    const int origin = block_origin(l, c, f, kappa);
    for_block_cells(origin, f, kappa, [&](int ss, int j) {
        if (!UNIFORM && ss != s) return;
        const double nuj = P.nu[j];
        double bj = 0.0;
        if (nuj > 0.0) {
            if (acc <= 0.0) r.zcol = 1;
            else bj = div_shared(nuj, acc, rcp);
            range_acc(bj, r.bmin, r.bmax, r.nonfinite);
            r.gap += fabs(__dsub_rn(nuj, __dmul_rn(bj, acc)));
        }
        P.b[j] = bj;
    });
}

// coarse block of fine cell i
__device__ __forceinline__ int block_of(int i, const G32 &f, const G32 &c, int kappa) {
    int k = 0;
    for (int a = f.nd - 1; a >= 0; --a) {
        const int x = i / f.stride[a];
        i -= x * f.stride[a];
        k += (x / kappa) * c.stride[a];
    }
    return k;
}

__global__ void block_map_kernel(G32 f, G32 c, int kappa, int32_t *__restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f.cells; i += gridDim.x * blockDim.x)
        out[i] = block_of(i, f, c, kappa);
}

// Uniform kernel, phase R cell work spread over every thread: with the
// block sums kb[] complete, a_next = mu / kb, the gap / range terms of the
// current a and the zero-row check (same arithmetic as row_unit's cell loop).
// (cells in groups of CP_U per thread: every independent load of a group is
// issued before its dependent gathers and arithmetic)
constexpr int CP_U = 8;

__device__ __forceinline__ void cell_pass_row(const PairPtrs &P, const G32 &f,
                                              const int32_t *__restrict__ bmap, bool init, const double *a_cur,
                                              double *a_next, Red &r, const double *kbs,
                                              const double *rcps) {
    for (int i0 = threadIdx.x; i0 < f.cells; i0 += PT * CP_U) {
        int kk[CP_U];
        double mu_[CP_U], ai_[CP_U], acc_[CP_U], rc_[CP_U];
#pragma unroll
        for (int q = 0; q < CP_U; ++q) {
            const int i = i0 + q * PT;
            const bool in = i < f.cells;
            kk[q] = in ? bmap[i] : 0;
            mu_[q] = in ? P.mu[i] : 0.0;
            ai_[q] = (in && !init) ? a_cur[i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < CP_U; ++q) {
            acc_[q] = kbs[kk[q]];
            rc_[q] = rcps[kk[q]];
        }
#pragma unroll
        for (int q = 0; q < CP_U; ++q) {
            const int i = i0 + q * PT;
            if (i >= f.cells) break;
            const double acc = acc_[q], mui = mu_[q];
            if (!init) {
                const double ai = ai_[q];
                range_acc(ai, r.amin, r.amax, r.nonfinite);
                if (mui > 0.0) r.gap += fabs(__dsub_rn(__dmul_rn(ai, acc), mui));
            }
            double an = 0.0;
            if (mui > 0.0) {
                if (acc <= 0.0) r.zrow = 1;
                else an = div_shared(mui, acc, rc_[q]);
            }
            a_next[i] = an;
        }
    }
}

__device__ __forceinline__ void cell_pass_col(const PairPtrs &P, const G32 &f,
                                              const int32_t *__restrict__ bmap, Red &r, const double *ktas,
                                              const double *rcps) {
    for (int j0 = threadIdx.x; j0 < f.cells; j0 += PT * CP_U) {
        int ll[CP_U];
        double nu_[CP_U], acc_[CP_U], rc_[CP_U];
#pragma unroll
        for (int q = 0; q < CP_U; ++q) {
            const int j = j0 + q * PT;
            const bool in = j < f.cells;
            ll[q] = in ? bmap[j] : 0;
            nu_[q] = in ? P.nu[j] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < CP_U; ++q) {
            acc_[q] = ktas[ll[q]];
            rc_[q] = rcps[ll[q]];
        }
#pragma unroll
        for (int q = 0; q < CP_U; ++q) {
            const int j = j0 + q * PT;
            if (j >= f.cells) break;
            const double acc = acc_[q], nuj = nu_[q];
            double bj = 0.0;
            if (nuj > 0.0) {
                if (acc <= 0.0) r.zcol = 1;
                else bj = div_shared(nuj, acc, rc_[q]);
                range_acc(bj, r.bmin, r.bmax, r.nonfinite);
                r.gap += fabs(__dsub_rn(nuj, __dmul_rn(bj, acc)));
            }
            P.b[j] = bj;
        }
    }
}

// The uniform kernel's walk of every row / column unit, once per launch:
// run r of arc q (CSR order) -> first fine cell, coefficient mass * W and
// product slot, one thread per ARC: the
// position of run (arc q, offsets s_{d-1..1}) in its unit's walk order follows
// from the coordinate groups q belongs to (per level the walk visits the
// groups of equal coarse coordinate in order and, inside a group, the kappa
// fine offsets one after the other), so a thread finds its arc's groups once
// (a scan over the unit's arcs) and then writes its K1 runs (the order
// `walk` enumerates: lexicographic over (l_{d-1}, s_{d-1}, ..., l_0)).
struct RunListArgs {  // one direction: CSR (rows) or CSC (columns) of the coarse plans
    const int32_t *ptr;
    const int64_t *pc;
    const double *mass;
    int32_t *cells;
    double *coefs;
    int32_t *dst;
};

__global__ void __launch_bounds__(128) run_list_par_kernel(
    const int64_t *__restrict__ arc_off, RunListArgs rows, RunListArgs cols,
    const double *__restrict__ W, int64_t batch, G32 f, G32 c, int kappa) {
    const RunListArgs &A = blockIdx.y == 0 ? rows : cols;
    const int32_t *__restrict__ ptr = A.ptr;
    const int64_t *__restrict__ pc = A.pc;
    const double *__restrict__ mass = A.mass;
    int32_t *__restrict__ cells = A.cells;
    double *__restrict__ coefs = A.coefs;
    int32_t *__restrict__ dst = A.dst;
    const int n = c.cells, nd = f.nd;
    const int K1 = (int)ipow(kappa, nd - 1);
    const double Wu = W[0];
    const int64_t total = arc_off[batch];
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        // pair of arc g: last b with arc_off[b] <= g
        int64_t blo = 0, bhi = batch - 1;
        while (blo < bhi) {
            const int64_t mid = (blo + bhi + 1) >> 1;
            if (arc_off[mid] <= g) blo = mid;
            else bhi = mid - 1;
        }
        const int64_t b = blo, a0 = arc_off[b];
        const int qa = (int)(g - a0);  // arc index inside the pair
        const int32_t *pp = ptr + b * (n + 1);
        if (qa >= pp[n]) continue;
        int ulo = 0, uhi = n - 1;  // unit of the arc: last u with ptr[u] <= qa
        while (ulo < uhi) {
            const int mid = (ulo + uhi + 1) >> 1;
            if (pp[mid] <= qa) ulo = mid;
            else uhi = mid - 1;
        }
        const int lo0 = pp[ulo], cnt = pp[ulo + 1] - lo0, q = qa - lo0;
        const int64_t *up = pc + a0 + lo0;
        int32_t *oc = cells + (a0 + lo0) * K1;
        double *of = coefs + (a0 + lo0) * K1;
        int32_t *od = dst + (a0 + lo0) * K1;
        // product slot of run `pos` of this unit in the cluster kernel's shared
        // buffer: chain order, each unit shifted by 2 doubles more than the one
        // before (CL_SKEW) so that the lanes of a warp, one chain each, read
        // different banks (unit sizes are multiples of 128 bytes)
        const int dbase = lo0 * K1 * kappa + CL_SKEW * ulo;
        const double cf = __dmul_rn(mass[a0 + qa], Wu);
        const int64_t w = up[q];
        // per level (d-1 .. 1): runs before the arc's group, the group's size,
        // the cell offset of the arc's coarse coordinate
        int before[GDT_MAX_DIM], gsize[GDT_MAX_DIM], cbase[GDT_MAX_DIM];
        int lo = 0, hi = cnt, kp = K1, pos0 = 0;
#pragma unroll
        for (int level = GDT_MAX_DIM - 1; level >= 1; --level) {
            if (level > nd - 1) continue;
            const int cr = pc_coord(w, level);
            int gs = q, ge = q + 1;
            while (gs > lo && pc_coord(up[gs - 1], level) == cr) --gs;
            while (ge < hi && pc_coord(up[ge], level) == cr) ++ge;
            pos0 += (gs - lo) * kp;
            kp /= kappa;  // runs per arc below this level
            before[level] = kp;
            gsize[level] = ge - gs;
            cbase[level] = cr * kappa;
            lo = gs;
            hi = ge;
        }
        pos0 += q - lo;
        const int cell0 = pc_coord(w, 0) * kappa;
        for (int r = 0; r < K1; ++r) {
            int rem = r, pos = pos0, cell = cell0;
#pragma unroll
            for (int level = GDT_MAX_DIM - 1; level >= 1; --level) {
                if (level > nd - 1) continue;
                const int sa = rem / before[level];
                rem -= sa * before[level];
                pos += sa * gsize[level] * before[level];
                cell += (cbase[level] + sa) * f.stride[level];
            }
            oc[pos] = cell;
            of[pos] = cf;
            od[pos] = dbase + pos * kappa;
        }
    }
}

// per-pair scalar record written by ipf_kernel / finish_kernel
// out[b*8 + {0..7}] = {transport_p, tv_mu, tv_nu, gap, iterations, converged, support, 0}

template <bool UNIFORM>
__global__ void __launch_bounds__(PT) ipf_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const int64_t *__restrict__ arc_off,
    const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ row_arc_col,
    const double *__restrict__ row_arc_mass, const int32_t *__restrict__ col_ptr,
    const int32_t *__restrict__ col_arc_row, const double *__restrict__ col_arc_mass,
    const double *__restrict__ W, const double *__restrict__ xi_in, int64_t max_iter, G32 f,
    G32 c, int kappa, double *__restrict__ out, int32_t *__restrict__ status,
    double *__restrict__ scratch, int64_t stride_pair, const int64_t *__restrict__ rpc,
    const int64_t *__restrict__ cpc, int use_smem, const int32_t *__restrict__ bmap,
    const int32_t *__restrict__ rl_cells, const double *__restrict__ rl_coef,
    const int32_t *__restrict__ cl_cells, const double *__restrict__ cl_coef, int prod_smem) {
    __shared__ double sh[(PT / 32 + 1) * 6];
    const int64_t b = blockIdx.x;
    const int N = f.cells, n = c.cells;
    const int m = (int)ipow(kappa, f.nd);
    const int U = UNIFORM ? n : N;
    const double Wu = W[0];

    PairPtrs P;
    P.mu = mu + b * N;
    P.nu = nu + b * N;
    const int64_t a0 = arc_off[b];
    P.rptr = row_ptr + b * (n + 1);
    P.cptr = col_ptr + b * (n + 1);
    P.rcol = row_arc_col + a0;
    P.rmass = row_arc_mass + a0;
    P.crow = col_arc_row + a0;
    P.cmass = col_arc_mass + a0;
    P.rpc = rpc + a0;
    P.cpc = cpc + a0;
    {
        const int64_t K1 = ipow(kappa, f.nd - 1);
        P.rrc = rl_cells ? rl_cells + a0 * K1 : nullptr;
        P.rrf = rl_coef ? rl_coef + a0 * K1 : nullptr;
        P.crc = cl_cells ? cl_cells + a0 * K1 : nullptr;
        P.crf = cl_coef ? cl_coef + a0 * K1 : nullptr;
    }
    P.pf = !use_smem;
    double *ws = scratch + b * stride_pair;
    P.aA = ws;
    P.aB = ws + N;
    P.b = ws + 2 * N;
    P.kb = ws + 3 * N;
    P.kta = ws + 3 * N + U;

    // supports and the reference's default xi (quantized.py:317-320)
    double cnt = 0.0;
    for (int i = threadIdx.x; i < N; i += PT) {
        const double mi = P.mu[i], ni = P.nu[i];
        cnt += (mi > 0.0 ? 1.0 : 0.0) + (ni > 0.0 ? 1.0 : 0.0);
        P.b[i] = ni > 0.0 ? 1.0 : 0.0;  // b = ones over the target support
    }
    cnt = block_sum<PT>(cnt, sh);
    const double xi = xi_in[b] < 0.0 ? 1e-9 * cnt : xi_in[b];
    __syncthreads();

    // The sequential exact-order sums of the long units are load-latency
    // bound; when the grid fits, the vector they gather from (b for row
    // units, a for column units) is staged in shared memory first.
    extern __shared__ double sx[];
    auto stage = [&](const double *src) -> const double * {
        if (!use_smem) return src;
        for (int i = threadIdx.x; i < N; i += PT) sx[i] = src[i];
        __syncthreads();
        return sx;
    };

    // kb = K b0, a = mu / kb (sinkhorn.py:119-129 before the first sweep)
    Red r = red_init();
    double *a_cur = P.aA, *a_nxt = P.aB;
    // uniform kernel: block sums, then per-block reciprocals, then the cell
    // work of the pass spread over all threads
    auto finish_units = [&](const double *sums, double *rcps) {
        __syncthreads();
        for (int u = threadIdx.x; u < U; u += PT) {
            const double v = sums[u];
            rcps[u] = v > 0.0 ? __drcp_rn(v) : 0.0;
        }
        __syncthreads();
    };
    double *rcp_buf = P.kta + U;  // scratch after kta (U doubles, see primal_layout)
    // two-phase unit sums (uniform kernel, kappa <= 8)
    // (products in shared memory after the staged vector, when the host sized
    // the dynamic shared memory for them: prod_smem != 0)
    const int K1 = UNIFORM ? (int)ipow(kappa, f.nd - 1) : 0;
    // prod_smem = doubles of shared memory for the products (0: off); they
    // follow the staged vector when it is staged, else start at offset 0
    double *prod = (UNIFORM && prod_smem > 0) ? sx + (use_smem ? ((N + 1) & ~1) : 0) : nullptr;
    const bool two_phase = UNIFORM && kappa <= 8 && prod != nullptr;
    if (two_phase) {  // the pair's CSR / CSC pointers in shared memory (after the products)
        int32_t *sp = reinterpret_cast<int32_t *>(prod + prod_smem);
        for (int i = threadIdx.x; i <= U; i += PT) {
            sp[i] = P.rptr[i];
            sp[U + 1 + i] = P.cptr[i];
        }
        P.rptr = sp;
        P.cptr = sp + U + 1;
        __syncthreads();
    }
    const double *bs = stage(P.b);
    if (two_phase) {
        unit_sums(P.rrc, P.rrf, P.rptr, U, K1, kappa, bs, prod, P.kb, prod_smem, P.pf);
    } else {
        for (int u = threadIdx.x; u < U; u += PT)
            row_unit<UNIFORM>(u, P, c, f, kappa, m, W, Wu, true, nullptr, a_cur, r, bs);
    }
    if (UNIFORM) {
        finish_units(P.kb, rcp_buf);
        cell_pass_row(P, f, bmap, true, nullptr, a_cur, r, P.kb, rcp_buf);
    }
    block_reduce_red(r, sh);
    int st = r.zrow ? GDT_PAIR_ZERO_DENOM_ROW : GDT_PAIR_OK;
    int64_t it = 0;
    double gap = INFINITY;
    bool converged = false;
    while (st == GDT_PAIR_OK && it < max_iter) {
        ++it;
        EX_TRACE(0);
        Red rc = red_init();
        const double *as = stage(a_cur);
        EX_TRACE(1);
        if (two_phase) unit_sums(P.crc, P.crf, P.cptr, U, K1, kappa, as, prod, P.kta, prod_smem, P.pf);
        else
            for (int u = threadIdx.x; u < U; u += PT)
                col_unit<UNIFORM>(u, P, c, f, kappa, m, W, Wu, a_cur, rc, as);
        EX_TRACE(2);
        if (UNIFORM) {
            finish_units(P.kta, rcp_buf);
            EX_TRACE(3);
            cell_pass_col(P, f, bmap, rc, P.kta, rcp_buf);
        }
        if (__syncthreads_or(rc.zcol)) {  // before anything reads b
            st = GDT_PAIR_ZERO_DENOM_COL;
            break;
        }
        EX_TRACE(4);
        const double *bsw = stage(P.b);
        EX_TRACE(5);
        if (two_phase) {
            __syncthreads();  // the column sums are done reading the product buffer
            unit_sums(P.rrc, P.rrf, P.rptr, U, K1, kappa, bsw, prod, P.kb, prod_smem, P.pf);
        } else {
            for (int u = threadIdx.x; u < U; u += PT)
                row_unit<UNIFORM>(u, P, c, f, kappa, m, W, Wu, false, a_cur, a_nxt, rc, bsw);
        }
        EX_TRACE(6);
        if (UNIFORM) {
            finish_units(P.kb, rcp_buf);
            EX_TRACE(7);
            cell_pass_row(P, f, bmap, false, a_cur, a_nxt, rc, P.kb, rcp_buf);
        }
        EX_TRACE(8);
        block_reduce_red(rc, sh);
        EX_TRACE(9);
        // _check_scale_range(a), then (b) (sinkhorn.py:137-138)
        const bool bad_a = rc.amin <= rc.amax &&
                           (rc.amin < 1e-100 || rc.amax > 1e100 || !isfinite(rc.amax));
        const bool bad_b = rc.bmin <= rc.bmax &&
                           (rc.bmin < 1e-100 || rc.bmax > 1e100 || !isfinite(rc.bmax));
        if (bad_a || bad_b || rc.nonfinite) {
            st = GDT_PAIR_OVERFLOW;
            break;
        }
        gap = rc.gap;
        if (gap < xi) {
            converged = true;
            break;
        }
        if (it >= max_iter) break;
        if (rc.zrow) {  // the check at the top of the next sweep
            st = GDT_PAIR_ZERO_DENOM_ROW;
            break;
        }
        double *tmp = a_cur;
        a_cur = a_nxt;
        a_nxt = tmp;
    }
    // publish which buffer holds the final a (aA or aB) for the pricing kernels
    if (threadIdx.x == 0) {
        status[b] = st;
        double *o = out + b * 8;
        o[0] = 0.0;
        o[1] = 0.0;
        o[2] = 0.0;
        o[3] = gap;
        o[4] = (double)it;
        o[5] = converged ? 1.0 : 0.0;
        o[6] = cnt;
        o[7] = a_cur == P.aA ? 0.0 : 1.0;
    }
}

// ---------------------------------------------------------------------------
// ipf_fast_kernel (fp32 mode, uniform kernel): the same sweep as ipf_kernel
// -- a = mu / K b, b = nu / K^T a, the reference's checks in its order
// (sinkhorn.py:119-141) -- with the block-sparse mat-vecs regrouped by the
// plan's block structure: with W_ts = W for every cell pair of an arc,
//   (K^T a)_s = sum_{k -> l(s)} m_kl W S_k,  S_k = sum_{t in X_k} a_t,
//   (K b)_t   = sum_{l <- k(t)} m_kl W B_l,  B_l = sum_{s in Y_l} b_s,
// so a sweep is two coalesced streaming passes over the fine cells (per
// coarse block: one thread, its kappa^d cells, the block sum in a register)
// and two O(arcs) passes over the coarse plan.  The summation order differs
// from scipy's CSR/CSC order (fp64 throughout, rounding-level differences;
// the fp32-mode contract is 1e-5 on the bounds), which removes the
// sequential per-unit chains whose length (up to m_kl * kappa^d terms) bounds
// ipf_kernel.  One thread-block cluster per pair (<= 8 CTAs), two cluster
// barriers per sweep; cross-CTA sums combine per-CTA partials in rank order
// (deterministic).
// Per sweep and fine cell: read mu, a, write a; read nu, write b = 40 bytes.
constexpr int FT = 256;  // threads per CTA of ipf_fast_kernel
constexpr int FCS_MAX = 8;

struct FastPart {
    double gap, lo, hi;
    int flags, pad;  // flags: 1 = zero denominator, 2 = non-finite
};

__device__ __forceinline__ FastPart fp_init() { return FastPart{0.0, INFINITY, -INFINITY, 0, 0}; }

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// address of the same shared variable in CTA `rank` of the cluster (DSMEM)
template <class T>
__device__ __forceinline__ T *dsmem(T *p, unsigned rank) {
    uint64_t out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
    return reinterpret_cast<T *>(out);
}

// CTA-reduce q into *mine (this CTA's shared slot, read by the cluster after
// the next cluster barrier)
__device__ __forceinline__ void fp_publish(FastPart q, FastPart *mine, FastPart *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        q.gap += __shfl_xor_sync(0xffffffffu, q.gap, o);
        q.lo = fmin(q.lo, __shfl_xor_sync(0xffffffffu, q.lo, o));
        q.hi = fmax(q.hi, __shfl_xor_sync(0xffffffffu, q.hi, o));
        q.flags |= __shfl_xor_sync(0xffffffffu, q.flags, o);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
        FastPart t = sh[0];
        for (int i = 1; i < FT / 32; ++i) {
            t.gap += sh[i].gap;
            t.lo = fmin(t.lo, sh[i].lo);
            t.hi = fmax(t.hi, sh[i].hi);
            t.flags |= sh[i].flags;
        }
        *mine = t;
    }
}

// after a cluster barrier: combine the cluster's slots in rank order (thread
// 0 reads them over DSMEM, the CTA shares the result through shared memory)
__device__ __forceinline__ FastPart fp_combine(FastPart *mine, unsigned cs, FastPart *sh) {
    if (threadIdx.x < 32) {
        // lane r reads CTA r's slot; lane 0 combines them in rank order
        const FastPart t = threadIdx.x < cs ? *dsmem(mine, threadIdx.x) : fp_init();
        FastPart o = fp_init();
        for (unsigned r = 0; r < cs; ++r) {
            o.gap += __shfl_sync(0xffffffffu, t.gap, r);
            o.lo = fmin(o.lo, __shfl_sync(0xffffffffu, t.lo, r));
            o.hi = fmax(o.hi, __shfl_sync(0xffffffffu, t.hi, r));
            o.flags |= __shfl_sync(0xffffffffu, t.flags, r);
        }
        if (threadIdx.x == 0) sh[FT / 32] = o;
    }
    __syncthreads();
    return sh[FT / 32];
}

__device__ __forceinline__ bool fp_bad(double lo, double hi) {
    return lo <= hi && (lo < 1e-100 || hi > 1e100 || !isfinite(hi));
}

// range and flags of mass / den over a block whose positive masses span
// [mlo, mhi] (mlo = +inf: no positive mass): correctly rounded division by a
// positive constant is monotone, so these are the min / max of the block's
// scalings; den <= 0 with positive mass is the zero-denominator case
__device__ __forceinline__ void fp_block_range(double mlo, double mhi, double den, double rcp,
                                               FastPart &q) {
    if (!(mlo <= mhi)) return;
    if (den <= 0.0) {
        q.flags |= 1;
        return;
    }
    const double lo = div_shared(mlo, den, rcp), hi = div_shared(mhi, den, rcp);
    if (isnan(lo) || isnan(hi) || !isfinite(hi)) q.flags |= 2;
    if (lo > 0.0) q.lo = fmin(q.lo, lo);
    if (hi > 0.0) q.hi = fmax(q.hi, hi);
}

// scaling of one cell: mass / den on the support, 0 elsewhere or when den <= 0.
// Markstein quotient without div_shared's range guards: correctly rounded
// whenever mass, den and the quotient stay inside the normal range, which the
// scale-range checks (1e-100 .. 1e100, evaluated with the guarded division on
// the block extremes) require of every accepted sweep anyway.
__device__ __forceinline__ double fp_scale(double m, double den, double rcp) {
    const double q = __dmul_rn(m, rcp);
    const double r = __fma_rn(-q, den, m);
    return (m > 0.0 && den > 0.0) ? __fma_rn(r, rcp, q) : 0.0;
}

__device__ __forceinline__ double fp_rcp(double den) { return den > 0.0 ? __drcp_rn(den) : 0.0; }

#ifdef GDT_IPF_TRACE
__device__ unsigned long long g_ipf_trace[128];
#define FP_TRACE(slot_)                                                                    \
    do {                                                                                   \
        if (blockIdx.x < 8 && threadIdx.x == 0 && it == 10) {                              \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
            g_ipf_trace[blockIdx.x * 16 + (slot_)] = t_;                                   \
        }                                                                                  \
    } while (0)
#else
#define FP_TRACE(slot_) \
    do {                \
    } while (0)
#endif

// Work mapping: a unit is one fine row (KAPPA cells along axis 0) of one
// coarse block; the G = kappa^(d-1) rows of a block sit in G consecutive
// lanes, which fold the block sum with xor shuffles (fixed order:
// deterministic).  KAPPA = 0: runtime kappa (or G > 32), one thread per
// block walking its rows.
template <int KAPPA>
__device__ __forceinline__ void fp_load(const double *p, double *v, int kappa) {
    if constexpr (KAPPA >= 2) {
#pragma unroll
        for (int x = 0; x < KAPPA; x += 2) {
            const double2 t = __ldg(reinterpret_cast<const double2 *>(p + x));
            v[x] = t.x;
            v[x + 1] = t.y;
        }
    } else {
        for (int x = 0; x < kappa; ++x) v[x] = __ldg(p + x);
    }
}

template <int KAPPA>
__device__ __forceinline__ void fp_store(double *p, const double *v, int kappa) {
    if constexpr (KAPPA >= 2) {
#pragma unroll
        for (int x = 0; x < KAPPA; x += 2)
            *reinterpret_cast<double2 *>(p + x) = make_double2(v[x], v[x + 1]);
    } else {
        for (int x = 0; x < kappa; ++x) p[x] = v[x];
    }
}

// xor-fold over the G lanes of a group (G warp-uniform, all lanes participate)
__device__ __forceinline__ double group_sum(double v, int G) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
        if (o < G) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Shared-memory plan of one CTA (byte offsets, 16-aligned):
//   src [n] f64      block sums of the whole pair gathered over DSMEM
//   own [2 nblk] f64 this CTA's block sums of a (S) and b (B), read remotely
//   blk [5 nblk] f64 per own block: min/max positive mu, min/max positive nu,
//                    and kb of the previous sweep (to recompute a)
//   kv  [2 nblk] f64 per own block: current kb and kta
//   rp/cp [nblk+1] i32 CSR / CSC pointer slices, rows [upc] i32 row starts
//   rc/cc [cap] f64 arc coefficients m W, ri/ci [cap] i32 arc endpoints,
//   prod [cap] f64 per-arc products of the current coarse pass
struct FpSmem {
    int src, own, blk, kv, rp, cp, rows, rc, ri, cc, ci, prod, total;
};

__host__ __device__ inline int fp_al(int x) { return (x + 15) & ~15; }

__host__ __device__ inline FpSmem fp_smem_plan(int n, int nblk, int upc, int cap) {
    FpSmem m;
    int o = 0;
    m.src = o;
    o = fp_al(o + 8 * n);
    m.own = o;
    o = fp_al(o + 16 * nblk);
    m.blk = o;
    o = fp_al(o + 40 * nblk);
    m.kv = o;
    o = fp_al(o + 16 * nblk);
    m.rp = o;
    o = fp_al(o + 4 * (nblk + 1));
    m.cp = o;
    o = fp_al(o + 4 * (nblk + 1));
    m.rows = o;
    o = fp_al(o + 4 * upc);
    m.rc = o;
    o = fp_al(o + 8 * cap);
    m.ri = o;
    o = fp_al(o + 4 * cap);
    m.cc = o;
    o = fp_al(o + 8 * cap);
    m.ci = o;
    o = fp_al(o + 4 * cap);
    m.prod = o;
    o = fp_al(o + 8 * cap);
    m.total = o;
    return m;
}

template <int KAPPA>
__global__ void __launch_bounds__(FT, 3) ipf_fast_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const int64_t *__restrict__ arc_off,
    const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ row_arc_col,
    const double *__restrict__ row_arc_mass, const int32_t *__restrict__ col_ptr,
    const int32_t *__restrict__ col_arc_row, const double *__restrict__ col_arc_mass,
    const double *__restrict__ W, const double *__restrict__ xi_in, int64_t max_iter, G32 f,
    G32 c, int kappa, double *__restrict__ out, int32_t *__restrict__ status,
    double *__restrict__ scratch, int64_t stride_pair, int cap) {
    constexpr int KV = KAPPA >= 2 ? KAPPA : 16;  // register row buffer (runtime kappa <= 16)
    // request a unit's masses before its coarse sum (kappa <= 4: the row
    // buffer fits the register budget next to the rest)
    constexpr bool EARLY = KAPPA >= 2 && KAPPA <= 4;
    __shared__ FastPart sh[FT / 32 + 1];
    __shared__ FastPart slot[3];  // this CTA's partials: init, row pass, column pass
    extern __shared__ __align__(16) unsigned char fsm[];
    const unsigned cs = cluster_size(), rank = cluster_rank_id();
    const int64_t b = blockIdx.x / cs;
    const int N = f.cells, n = c.cells;
    const double Wu = W[0];
    const double *mub = mu + b * N, *nub = nu + b * N;
    const int64_t a0 = arc_off[b];
    const int32_t *rptr = row_ptr + b * (n + 1), *cptr = col_ptr + b * (n + 1);
    const int32_t *rcol = row_arc_col + a0, *crow = col_arc_row + a0;
    const double *rmass = row_arc_mass + a0, *cmass = col_arc_mass + a0;
    double *ws = scratch + b * stride_pair;
    double *aA = ws, *bv = ws + 2 * N, *kbv = ws + 3 * N, *ktv = ws + 3 * N + n;
    const int kp = KAPPA >= 2 ? KAPPA : kappa;
    int rows = 1;  // fine rows per block
    for (int a = 1; a < f.nd; ++a) rows *= kp;
    const int G = KAPPA >= 2 ? rows : 1;           // lanes per block
    const int rows_per_unit = KAPPA >= 2 ? 1 : rows;
    const int units = n * G;
    // CTA `rank` owns a contiguous, warp-aligned range of units (so its blocks
    // are contiguous too); trip counts are CTA-uniform (shuffles need every lane)
    const int upc = (((units + (int)cs - 1) / (int)cs) + 31) / 32 * 32;
    const int bpc = upc / G;  // blocks per CTA (owner of block k: k / bpc)
    const int u_lo = (int)rank * upc;
    const int trips = (upc + FT - 1) / FT;
    const int k_lo = min((int)rank * bpc, n);
    const int nblk = max(0, min(bpc, n - k_lo));
    const int r_lo = rptr[k_lo], r_n = rptr[k_lo + nblk] - r_lo;
    const int c_lo = cptr[k_lo], c_n = cptr[k_lo + nblk] - c_lo;
    const bool arcs_s = r_n <= cap && c_n <= cap;
    const FpSmem L = fp_smem_plan(n, bpc, upc, cap);
    double *src_s = reinterpret_cast<double *>(fsm + L.src);
    double *ownS = reinterpret_cast<double *>(fsm + L.own), *ownB = ownS + bpc;
    double *blk_s = reinterpret_cast<double *>(fsm + L.blk);  // [bpc][5]
    double *kb_s = reinterpret_cast<double *>(fsm + L.kv), *kt_s = kb_s + bpc;
    int *rp_s = reinterpret_cast<int *>(fsm + L.rp), *cp_s = reinterpret_cast<int *>(fsm + L.cp);
    int *row_s = reinterpret_cast<int *>(fsm + L.rows);
    double *rc_s = reinterpret_cast<double *>(fsm + L.rc), *cc_s = reinterpret_cast<double *>(fsm + L.cc);
    int *ri_s = reinterpret_cast<int *>(fsm + L.ri), *ci_s = reinterpret_cast<int *>(fsm + L.ci);
    double *prod_s = reinterpret_cast<double *>(fsm + L.prod);

    // ---- per-CTA tables (once) ----
    for (int i = threadIdx.x; i <= nblk; i += FT) {
        rp_s[i] = rptr[k_lo + i] - r_lo;
        cp_s[i] = cptr[k_lo + i] - c_lo;
    }
    if (arcs_s) {
        for (int e = threadIdx.x; e < r_n; e += FT) {
            rc_s[e] = __dmul_rn(rmass[r_lo + e], Wu);
            ri_s[e] = rcol[r_lo + e];
        }
        for (int e = threadIdx.x; e < c_n; e += FT) {
            cc_s[e] = __dmul_rn(cmass[c_lo + e], Wu);
            ci_s[e] = crow[c_lo + e];
        }
    }
    for (int i = threadIdx.x; i < upc; i += FT) {
        const int u = u_lo + i;
        int off = 0;
        if (u < units) {
            const int k = u / G;
            int q = u - k * G;
            off = block_origin(k, c, f, kp);
            for (int a = 1; a < f.nd && KAPPA >= 2; ++a) {
                off += (q % kp) * f.stride[a];
                q /= kp;
            }
        }
        row_s[i] = off;
    }
    for (int i = threadIdx.x; i < 5 * bpc; i += FT) {
        const int w = i % 5;
        blk_s[i] = w == 4 ? 0.0 : ((w & 1) ? -INFINITY : INFINITY);
    }
    __syncthreads();

    auto row_index = [&](int ui, int qq) {
        if constexpr (KAPPA >= 2) {
            return row_s[ui];
        } else {
            int off = 0, z = qq;
            for (int a = 1; a < f.nd; ++a) {
                off += (z % kp) * f.stride[a];
                z /= kp;
            }
            return row_s[ui] + off;
        }
    };
    // the pair's block sums (a: own = ownS, b: own = ownB) into src_s over DSMEM
    auto gather = [&](double *own) {
        for (int i = threadIdx.x; i < n; i += FT) {
            const unsigned r = (unsigned)(i / bpc);
            src_s[i] = *dsmem(own + (i - (int)r * bpc), r);
        }
        __syncthreads();
    };
    // per-arc products coef * src[endpoint] of this CTA's arcs, then each
    // block's G lanes add its arcs (fixed order)
    auto products = [&](const double *coef_s, const int *idx_s, int count) {
        if (arcs_s)
            for (int e = threadIdx.x; e < count; e += FT) prod_s[e] = coef_s[e] * src_s[idx_s[e]];
        __syncthreads();
    };
    auto coarse = [&](int k, int r, bool act, const int *ptr_s, int e_base, const int32_t *idx,
                      const double *mass) {
        double v = 0.0;
        if (act) {
            const int e0 = ptr_s[k - k_lo], e1 = ptr_s[k - k_lo + 1];
            if (arcs_s) {
                for (int e = e0 + r; e < e1; e += G) v += prod_s[e];
            } else {
                for (int e = e0 + r; e < e1; e += G)
                    v += __dmul_rn(__ldg(mass + e_base + e), Wu) * src_s[__ldg(idx + e_base + e)];
            }
        }
        return group_sum(v, G);
    };

    // b = 1 on the target support (sinkhorn.py:119 on the restricted matrix),
    // B_l = its count, support count for the default xi, block mass ranges
    {
        FastPart q = fp_init();
        for (int t = 0; t < trips; ++t) {
            const int ui = t * FT + (int)threadIdx.x, u = u_lo + ui;
            const bool act = u < units && ui < upc;
            const int l = act ? u / G : k_lo, r = act ? u - l * G : 0;
            double sb = 0.0, mlo = INFINITY, mhi = -INFINITY, nlo = INFINITY, nhi = -INFINITY;
            if (act)
                for (int qq = 0; qq < rows_per_unit; ++qq) {
                    const int j0 = row_index(ui, qq);
                    double nv[KV], mv[KV];
                    fp_load<KAPPA>(nub + j0, nv, kp);
                    fp_load<KAPPA>(mub + j0, mv, kp);
#pragma unroll
                    for (int x = 0; x < KV; ++x) {
                        if (x >= kp) break;
                        q.gap += (mv[x] > 0.0 ? 1.0 : 0.0) + (nv[x] > 0.0 ? 1.0 : 0.0);
                        sb += nv[x] > 0.0 ? 1.0 : 0.0;
                        if (mv[x] > 0.0) {
                            mlo = fmin(mlo, mv[x]);
                            mhi = fmax(mhi, mv[x]);
                        }
                        if (nv[x] > 0.0) {
                            nlo = fmin(nlo, nv[x]);
                            nhi = fmax(nhi, nv[x]);
                        }
                    }
                }
            sb = group_sum(sb, G);
            for (int o = 1; o < 32; o <<= 1)
                if (o < G) {
                    mlo = fmin(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
                    mhi = fmax(mhi, __shfl_xor_sync(0xffffffffu, mhi, o));
                    nlo = fmin(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
                    nhi = fmax(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
                }
            if (act && r == 0) {
                ownB[l - k_lo] = sb;
                double *bk = blk_s + 5 * (l - k_lo);
                bk[0] = mlo;
                bk[1] = mhi;
                bk[2] = nlo;
                bk[3] = nhi;
            }
        }
        fp_publish(q, &slot[0], sh);
    }
    cluster_sync_all();
    const double cnt = fp_combine(&slot[0], cs, sh).gap;
    const double xi = xi_in[b] < 0.0 ? 1e-9 * cnt : xi_in[b];

    int st = GDT_PAIR_OK;
    int64_t it = 0;
    bool converged = false;
    double gap = INFINITY;
    FastPart ra = fp_init(), rb = ra;  // a and b of sweep `it`
    for (;;) {
        // kb = K b (coarse); row pass: a of sweep it recomputed from its kb
        // (blk[4]) for |a kb - mu|, the zero-row check, a of sweep it+1 and
        // its block sums.  a is not stored: the closing pass writes the final one.
        FastPart q = fp_init();
        FP_TRACE(0);
        gather(ownB);
        FP_TRACE(1);
        products(rc_s, ri_s, r_n);
        FP_TRACE(2);
        for (int t = 0; t < trips; ++t) {
            const int ui = t * FT + (int)threadIdx.x, u = u_lo + ui;
            const bool act = u < units && ui < upc;
            const int k = act ? u / G : k_lo, r = act ? u - k * G : 0;
            // the unit's masses are requested first: their latency overlaps
            // the coarse sum and the reciprocals
            double mv0[KV];
            if (EARLY && act) fp_load<KAPPA>(mub + row_s[ui], mv0, kp);
            const double kb = coarse(k, r, act, rp_s, r_lo, rcol, rmass);
            const double rcp = fp_rcp(kb);
            double *bk = blk_s + 5 * (k - k_lo);
            const double kbo = act ? bk[4] : 0.0, rcpo = fp_rcp(kbo);
            double sa = 0.0;
            if (act) {
                if (r == 0) fp_block_range(bk[0], bk[1], kb, rcp, q);
                for (int qq = 0; qq < rows_per_unit; ++qq) {
                    double mv[KV];
                    if constexpr (EARLY) {
#pragma unroll
                        for (int x = 0; x < KV; ++x) mv[x] = mv0[x];
                    } else {
                        fp_load<KAPPA>(mub + row_index(ui, qq), mv, kp);
                    }
#pragma unroll
                    for (int x = 0; x < KV; ++x) {
                        if (x >= kp) break;
                        const double mi = mv[x];
                        if (it >= 1 && mi > 0.0) {
                            const double ao = fp_scale(mi, kbo, rcpo);
                            q.gap += fabs(__dsub_rn(__dmul_rn(ao, kb), mi));
                        }
                        sa += fp_scale(mi, kb, rcp);
                    }
                }
            }
            sa = group_sum(sa, G);
            if (act && r == 0) {
                ownS[k - k_lo] = sa;
                kb_s[k - k_lo] = kb;
            }
        }
        FP_TRACE(3);
        fp_publish(q, &slot[1], sh);
        FP_TRACE(4);
        cluster_sync_all();
        FP_TRACE(5);
        const FastPart ac = fp_combine(&slot[1], cs, sh);
        FP_TRACE(6);
        if (it >= 1) {  // end of sweep `it`: range checks, then the gap
            if (fp_bad(ra.lo, ra.hi) || fp_bad(rb.lo, rb.hi) || ((ra.flags | rb.flags) & 2)) {
                st = GDT_PAIR_OVERFLOW;
                break;
            }
            gap = ac.gap + rb.gap;
            if (gap < xi) {
                converged = true;
                break;
            }
            if (it >= max_iter) break;
        }
        if (ac.flags & 1) {  // top of sweep it+1
            st = GDT_PAIR_ZERO_DENOM_ROW;
            break;
        }
        ++it;
        ra = ac;
        // the kb that defines a of sweep `it` (kept for the recompute)
        for (int i = threadIdx.x; i < nblk; i += FT) blk_s[5 * i + 4] = kb_s[i];
        // kta = K^T a (coarse); column pass: zero-column check, b, |nu - b kta|,
        // range(b), block sums of b (b is not stored either)
        FastPart qb = fp_init();
        gather(ownS);
        FP_TRACE(7);
        products(cc_s, ci_s, c_n);
        FP_TRACE(8);
        for (int t = 0; t < trips; ++t) {
            const int ui = t * FT + (int)threadIdx.x, u = u_lo + ui;
            const bool act = u < units && ui < upc;
            const int l = act ? u / G : k_lo, r = act ? u - l * G : 0;
            double nv0[KV];
            if (EARLY && act) fp_load<KAPPA>(nub + row_s[ui], nv0, kp);
            const double kt = coarse(l, r, act, cp_s, c_lo, crow, cmass);
            const double rcp = fp_rcp(kt);
            double sb = 0.0;
            if (act) {
                if (r == 0) {
                    const double *bl = blk_s + 5 * (l - k_lo);
                    fp_block_range(bl[2], bl[3], kt, rcp, qb);
                }
                for (int qq = 0; qq < rows_per_unit; ++qq) {
                    double nv[KV];
                    if constexpr (EARLY) {
#pragma unroll
                        for (int x = 0; x < KV; ++x) nv[x] = nv0[x];
                    } else {
                        fp_load<KAPPA>(nub + row_index(ui, qq), nv, kp);
                    }
#pragma unroll
                    for (int x = 0; x < KV; ++x) {
                        if (x >= kp) break;
                        const double nj = nv[x];
                        const double v = fp_scale(nj, kt, rcp);
                        if (nj > 0.0) qb.gap += fabs(__dsub_rn(nj, __dmul_rn(v, kt)));
                        sb += v;
                    }
                }
            }
            sb = group_sum(sb, G);
            if (act && r == 0) {
                ownB[l - k_lo] = sb;
                kt_s[l - k_lo] = kt;
            }
        }
        FP_TRACE(9);
        fp_publish(qb, &slot[2], sh);
        FP_TRACE(10);
        cluster_sync_all();
        FP_TRACE(11);
        rb = fp_combine(&slot[2], cs, sh);
        FP_TRACE(12);
        if (rb.flags & 1) {
            st = GDT_PAIR_ZERO_DENOM_COL;
            break;
        }
    }
    // closing pass: the final a (from its kb, blk[4]) and b (from kta of the
    // same sweep) for pricing and TV, with kb = K b and kta = K^T a
    if (st == GDT_PAIR_OK && it >= 1) {
        __syncthreads();
        for (int t = 0; t < trips; ++t) {
            const int ui = t * FT + (int)threadIdx.x, u = u_lo + ui;
            if (u >= units || ui >= upc) continue;
            const int k = u / G, r = u - k * G;
            const double kbo = blk_s[5 * (k - k_lo) + 4], rcpo = fp_rcp(kbo);
            const double kt = kt_s[k - k_lo], rcpt = fp_rcp(kt);
            for (int qq = 0; qq < rows_per_unit; ++qq) {
                const int i0 = row_index(ui, qq);
                double mv[KV], nv[KV];
                fp_load<KAPPA>(mub + i0, mv, kp);
                fp_load<KAPPA>(nub + i0, nv, kp);
#pragma unroll
                for (int x = 0; x < KV; ++x) {
                    if (x >= kp) break;
                    mv[x] = fp_scale(mv[x], kbo, rcpo);
                    nv[x] = fp_scale(nv[x], kt, rcpt);
                }
                fp_store<KAPPA>(aA + i0, mv, kp);
                fp_store<KAPPA>(bv + i0, nv, kp);
            }
            if (r == 0) {
                kbv[k] = kb_s[k - k_lo];
                ktv[k] = kt;
            }
        }
    }
    cluster_sync_all();  // no CTA leaves while its shared memory may be read
    if (rank == 0 && threadIdx.x == 0) {
        status[b] = st;
        double *o = out + b * 8;
        o[0] = 0.0;
        o[1] = 0.0;
        o[2] = 0.0;
        o[3] = gap;
        o[4] = (double)it;
        o[5] = converged ? 1.0 : 0.0;
        o[6] = cnt;
        o[7] = 0.0;  // final a in the first buffer
    }
}

__device__ __forceinline__ float sqrt_apx32(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ double tv_weight(int i, const G32 &f, double p) {
    double parts[GDT_MAX_DIM];
    for (int a = f.nd - 1; a >= 0; --a) {
        const int x = i / f.stride[a];
        i -= x * f.stride[a];
        const double df = __dsub_rn((double)(x + 1), ((double)f.n[a] + 1.0) / 2.0);
        parts[a] = __dmul_rn(df, df);
    }
    double sq = -0.0;
    for (int a = 0; a < f.nd; ++a) sq = __dadd_rn(sq, parts[a]);
    if (p == 2.0) return sq;
    if (p == 1.0) return __dsqrt_rn(sq);
    return pow(sq, p / 2.0);
}

constexpr int MT = 128;  // threads of the moments/price kernels

// Per block: TV partials (per CTA) and moments of a and b about the block
// centre: mom[(b*n + k)*MW + {A0, A1[d], A2, B0, B1[d], B2}].
// ND / KAP > 0: compile-time dimension and pooling factor (the cell index
// arithmetic becomes shifts, the moment arrays stay in registers); 0 = runtime.
// tv_w: the padded grid's tv_weights table (host-computed with the
// reference's formula, measures.py:289-296) or NULL (computed per cell).
template <bool UNIFORM, int ND, int KAP>
__global__ void __launch_bounds__(MT) moments_tv_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const double *__restrict__ out,
    const int32_t *__restrict__ status, double *__restrict__ scratch, int64_t stride_pair,
    double *__restrict__ mom, double *__restrict__ part, G32 f, G32 c, int kappa_rt, double p,
    int want_moments, int lb, const double *__restrict__ tv_w) {
    const int kappa = KAP ? KAP : kappa_rt;
    const int nd = ND ? ND : f.nd;
    // one group of `lb` consecutive lanes per coarse block (tv_lanes: a power
    // of two dividing kappa^d): lane j of the group takes the block's cells
    // j, j + lb, ...; moments fold over the group by shuffles, TV partials
    // over the CTA (fixed order: deterministic)
    __shared__ double sh[32];
    const int64_t b = blockIdx.y;
    const int N = f.cells, n = c.cells;
    const int m = (int)ipow(kappa, nd);
    const int U = UNIFORM ? n : N;
    const int MW = 2 * (nd + 2);
    const int gid = blockIdx.x * MT + threadIdx.x;
    const int k = gid / lb, j = gid - k * lb;
    double tmu = 0.0, tnu = 0.0;
    double A[2 + GDT_MAX_DIM] = {0, 0, 0, 0, 0, 0}, Bm[2 + GDT_MAX_DIM] = {0, 0, 0, 0, 0, 0};
    const bool live = status[b] == GDT_PAIR_OK && k < n;
    if (live) {
        const double *ws = scratch + b * stride_pair;
        const double *a = out[b * 8 + 7] == 0.0 ? ws : ws + N;
        const double *bv = ws + 2 * N, *kb = ws + 3 * N, *kta = ws + 3 * N + U;
        const double *mub = mu + b * N, *nub = nu + b * N;
        const double ctr = (kappa - 1) / 2.0;
        const int origin = block_origin(k, c, f, kappa);
        for (int t = j; t < m; t += lb) {
            int i = origin, rem = t;
            double dl[GDT_MAX_DIM], r2 = 0.0;
#pragma unroll
            for (int q = 0; q < (ND ? ND : GDT_MAX_DIM); ++q) {
                if (q >= nd) break;
                const int o = rem % kappa;
                rem /= kappa;
                i += o * f.stride[q];
                dl[q] = (double)o - ctr;
                r2 += dl[q] * dl[q];
            }
            const double w = tv_w ? __ldg(tv_w + i) : tv_weight(i, f, p);
            const double kbu = kb[UNIFORM ? k : k * m + t];
            const double ktu = kta[UNIFORM ? k : k * m + t];
            const double ai = a[i], bi = bv[i];
            const double mh = mub[i] > 0.0 ? __dmul_rn(ai, kbu) : 0.0;
            const double nh = nub[i] > 0.0 ? __dmul_rn(bi, ktu) : 0.0;
            tmu += w * fabs(__dsub_rn(mh, mub[i]));
            tnu += w * fabs(__dsub_rn(nh, nub[i]));
            if (want_moments) {
#pragma unroll
                for (int q = 0; q < (ND ? ND : GDT_MAX_DIM); ++q) {
                    if (q >= nd) break;
                    A[1 + q] += ai * dl[q];
                    Bm[1 + q] += bi * dl[q];
                }
                A[0] += ai;
                Bm[0] += bi;
                A[1 + GDT_MAX_DIM] += ai * r2;
                Bm[1 + GDT_MAX_DIM] += bi * r2;
            }
        }
    }
    if (want_moments) {  // uniform across the CTA: every lane takes part in the shuffles
#pragma unroll
        for (int q = 0; q < 2 + GDT_MAX_DIM; ++q)
            for (int o = 1; o < lb; o <<= 1) {
                A[q] += __shfl_xor_sync(0xffffffffu, A[q], o, lb);
                Bm[q] += __shfl_xor_sync(0xffffffffu, Bm[q], o, lb);
            }
        if (live && j == 0) {
            double *o = mom + ((int64_t)b * n + k) * MW;
            // slots: A0, A1[nd], A2, then B likewise (second moments kept in the last register slot)
#pragma unroll
            for (int q = 0; q < 1 + GDT_MAX_DIM; ++q) {
                if (q > nd) break;
                o[q] = A[q];
                o[nd + 2 + q] = Bm[q];
            }
            o[nd + 1] = A[1 + GDT_MAX_DIM];
            o[2 * nd + 3] = Bm[1 + GDT_MAX_DIM];
        }
    }
    tmu = block_sum<MT>(tmu, sh);
    tnu = block_sum<MT>(tnu, sh);
    if (threadIdx.x == 0) {
        double *pp = part + ((int64_t)b * gridDim.x + blockIdx.x) * 2;
        pp[0] = tmu;
        pp[1] = tnu;
    }
}

// Per arc pricing.  p == 2 and uniform W: closed form from the block moments,
//   sum_{t,s} a_t b_s |D + d_t - e_s|^2 = A0 B0 |D|^2 + 2 D.(A1 B0 - A0 B1)
//                                          + A2 B0 + A0 B2 - 2 A1.B1,
// D = kappa (k - l); otherwise direct summation over the kappa^2d entries.
template <bool UNIFORM>
__global__ void __launch_bounds__(MT) price_kernel(
    const int64_t *__restrict__ arc_off, const int32_t *__restrict__ row_ptr,
    const int32_t *__restrict__ row_arc_col, const double *__restrict__ row_arc_mass,
    const double *__restrict__ W, const double *__restrict__ out, const int32_t *__restrict__ status,
    const double *__restrict__ scratch, int64_t stride_pair, const double *__restrict__ mom,
    double *__restrict__ part, G32 f, G32 c, int kappa, double p, const double *__restrict__ table,
    int closed_form, int fast, const int32_t *__restrict__ arc_row) {
    __shared__ double sh[32];
    const int64_t b = blockIdx.y;
    const int N = f.cells, n = c.cells;
    const int m = (int)ipow(kappa, f.nd);
    const int MW = 2 * (f.nd + 2);
    const int64_t A = arc_off[b + 1] - arc_off[b];
    double acc = 0.0;
    const int64_t item = (int64_t)blockIdx.x * MT + threadIdx.x;
    const int64_t q = closed_form ? item : item / m;       // arc
    const int t = closed_form ? 0 : (int)(item - q * m);   // row offset (brute force)
    if (status[b] == GDT_PAIR_OK && q < A) {
        int k;  // row block of arc q
        if (arc_row) {
            k = arc_row[arc_off[b] + q];
        } else {
            const int32_t *rptr = row_ptr + b * (n + 1);
            int lo = 0, hi = n;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (rptr[mid] <= q) lo = mid;
                else hi = mid;
            }
            k = lo;
        }
        const int l = row_arc_col[arc_off[b] + q];
        const double mass = row_arc_mass[arc_off[b] + q];
        if (closed_form) {
            const double *Ak = mom + ((int64_t)b * n + k) * MW;
            const double *Bl = mom + ((int64_t)b * n + l) * MW + (f.nd + 2);
            double d2 = 0.0, cross = 0.0, ab = 0.0;
            int kk = k, ll = l;
            for (int a = c.nd - 1; a >= 0; --a) {
                const int ka = kk / c.stride[a], la = ll / c.stride[a];
                kk -= ka * c.stride[a];
                ll -= la * c.stride[a];
                const double D = (double)(kappa * (ka - la));
                d2 += D * D;
                cross += D * (Ak[1 + a] * Bl[0] - Ak[0] * Bl[1 + a]);
                ab += Ak[1 + a] * Bl[1 + a];
            }
            const double s = Ak[0] * Bl[0] * d2 + 2.0 * cross + Ak[1 + f.nd] * Bl[0] +
                             Ak[0] * Bl[1 + f.nd] - 2.0 * ab;
            acc = mass * W[0] * s;
        } else {
            const double *ws = scratch + b * stride_pair;
            const double *a = out[b * 8 + 7] == 0.0 ? ws : ws + N;
            const double *bv = ws + 2 * N;
            // coordinates of row cell (k, t) minus the origin of block l
            int dd[GDT_MAX_DIM] = {0, 0, 0, 0};
            int i = 0, kk = k, ll = l, tt = t;
            for (int aa = c.nd - 1; aa >= 0; --aa) {
                const int ka = kk / c.stride[aa], la = ll / c.stride[aa];
                kk -= ka * c.stride[aa];
                ll -= la * c.stride[aa];
                dd[aa] = (ka - la) * kappa;
            }
            for (int aa = 0; aa < f.nd; ++aa) {
                const int ta = tt % kappa;
                tt /= kappa;
                dd[aa] += ta;
            }
            i = block_origin(k, c, f, kappa);
            {
                int rem = t;
                for (int aa = 0; aa < f.nd; ++aa) {
                    i += (rem % kappa) * f.stride[aa];
                    rem /= kappa;
                }
            }
            const double ai = a[i];
            if (ai != 0.0) {
                const double am = __dmul_rn(mass, UNIFORM ? W[0] : 0.0);
                const int ol = block_origin(l, c, f, kappa);
                // target cells of block l in ascending order with their squared
                // offsets kept incrementally (no per-cell division)
                const int K1 = f.nd > 1 ? kappa : 1, K2 = f.nd > 2 ? kappa : 1;
                int s = 0;
                for (int o2 = 0; o2 < K2; ++o2) {
                    const int e2 = f.nd > 2 ? dd[2] - o2 : 0;
                    for (int o1 = 0; o1 < K1; ++o1) {
                        const int e1 = f.nd > 1 ? dd[1] - o1 : 0;
                        const int hsq = e1 * e1 + e2 * e2;
                        const int row = ol + o2 * (f.nd > 2 ? f.stride[2] : 0) +
                                        o1 * (f.nd > 1 ? f.stride[1] : 0);
                        for (int o0 = 0; o0 < kappa; ++o0, ++s) {
                            const int e0 = dd[0] - o0;
                            const int sq = hsq + e0 * e0;
                            const double coef = UNIFORM ? am : __dmul_rn(mass, W[t * m + s]);
                            const double fitted = __dmul_rn(__dmul_rn(ai, coef), bv[row + o0]);
                            double cost;
                            if (p == 2.0) cost = (double)sq;
                            else if (fast && p == 1.0) cost = (double)sqrt_apx32((float)sq);
                            else cost = __ldg(table + sq);
                            acc += fitted * cost;
                        }
                    }
                }
            }
        }
    }
    acc = block_sum<MT>(acc, sh);
    if (threadIdx.x == 0) part[(int64_t)b * gridDim.x + blockIdx.x] = acc;
}

// row block of every arc (CSR order), for the pricing kernel
__global__ void arc_rows_kernel(const int64_t *__restrict__ arc_off,
                                const int32_t *__restrict__ row_ptr, int64_t batch, int n,
                                int32_t *__restrict__ arc_row) {
    const int64_t total = batch * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / n;
        const int k = (int)(i - b * n);
        const int32_t *rp = row_ptr + b * (n + 1);
        for (int e = rp[k]; e < rp[k + 1]; ++e) arc_row[arc_off[b] + e] = k;
    }
}

// one warp per pair: lanes stride over the CTA partials, fixed-order butterfly
__global__ void finish_kernel(const double *__restrict__ tv_part, int tv_ctas,
                              const double *__restrict__ pr_part, int pr_ctas,
                              const int32_t *__restrict__ status, double *__restrict__ out,
                              int64_t batch) {
    const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= batch || status[b] != GDT_PAIR_OK) return;  // warp-uniform
    double tmu = 0.0, tnu = 0.0, pr = 0.0;
    for (int i = lane; i < tv_ctas; i += 32) {
        tmu += tv_part[(b * tv_ctas + i) * 2];
        tnu += tv_part[(b * tv_ctas + i) * 2 + 1];
    }
    if (pr_part)
        for (int i = lane; i < pr_ctas; i += 32) pr += pr_part[b * pr_ctas + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tmu += __shfl_xor_sync(0xffffffffu, tmu, o);
        tnu += __shfl_xor_sync(0xffffffffu, tnu, o);
        pr += __shfl_xor_sync(0xffffffffu, pr, o);
    }
    if (lane == 0) {
        if (pr_part) out[b * 8 + 0] = pr;  // else the caller's kernel priced already
        out[b * 8 + 1] = tmu;
        out[b * 8 + 2] = tnu;
    }
}

// ---------------------------------------------------------------------------
// ipf_cluster_kernel: the exact-order IPF of ipf_kernel<true> (uniform kernel,
// two-phase unit sums) with one thread-block CLUSTER per pair.
//
// One CTA per pair left most of the GPU idle at the benchmark batch sizes
// (64 CTAs at cfg5, 45 at cfg3) and forced the products of a direction through
// several shared-memory batches, whose longest chains then ran one after the
// other.  Here rank r of the cluster owns a contiguous range of row units and
// of column units (balanced by arc count) and a contiguous slice of the fine
// cells.  Every unit is still summed by ONE thread over its products in the
// reference's order -- the bits of kb / kta, a and b do not depend on the
// cluster size -- only units and cells are spread over more SMs.  The vectors
// a, b, kb, kta live in global memory (L2); four cluster barriers per sweep
// order the phases (release/acquire at cluster scope, so plain loads after a
// barrier see the other CTAs' stores):
//     col sums | B | col cells (b, zero-column flag) | C | row sums | D |
//     row cells (next a, gap / range partials) | A: fold of the per-CTA
//     records in rank order, the reference's checks (sinkhorn.py:125-141)
// Every CTA takes the same decisions from the same folded record.
// ---------------------------------------------------------------------------

// loads of data another CTA of the cluster wrote before the last barrier:
// explicit ld.global (never the non-coherent path), issue order kept
__device__ __forceinline__ double ld_gl(const double *p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_gl2(const double *p) {
    double2 v;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

#ifdef GDT_IPF_TRACE
// debug builds: clocks inside the first unit-sum batch of the traced sweep (CTA 0)
__device__ int g_cl_on;
#define CL_TRACE(slot_)                                                                   \
    do {                                                                                  \
        if (blockIdx.x == 0 && threadIdx.x == 0 && g_cl_on == 1 && u0 == ua)              \
            g_ex_trace[8 + (slot_)] = clock64();                                          \
    } while (0)
#else
#define CL_TRACE(slot_) \
    do {                \
    } while (0)
#endif

// products of `nruns` runs (KAP cells each) in chain order into shared memory;
// RU runs per thread in flight (descriptors, then gathers, then products)
// The gathers go through cp.async (16-byte copies global -> shared, L2 path:
// coherent with the other CTAs' stores, and no register or scoreboard holds a
// copy in flight), so a thread keeps all its runs' gathers outstanding at
// once; the per-SM count of loads in flight, not the chains, bounded the
// register-staged version.  Each thread then scales the runs it fetched by
// their coefficients in place (same products, same slots).
__device__ __forceinline__ void cp_async16(double *smem_dst, const double *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}

template <int KAP>
__device__ __forceinline__ void cl_products(const int32_t *__restrict__ cells,
                                            const double *__restrict__ coefs,
                                            const int32_t *__restrict__ dst, int dbase, int nruns,
                                            const double *x, double *prod) {
    // an item is one 16-byte chunk (2 cells) of a run; consecutive threads take
    // consecutive chunks, so the KAP / 2 copies of a run sit in adjacent lanes
    // and share their cache line
    constexpr int CH = KAP / 2, IU = 8;
    const int nitems = nruns * CH;
    for (int t0 = threadIdx.x; t0 < nitems; t0 += PT * IU) {
        int cl[IU], ds[IU];
#pragma unroll
        for (int q = 0; q < IU; ++q) {
            const int t = t0 + q * PT, r = t / CH;
            cl[q] = t < nitems ? __ldg(cells + r) + 2 * (t - r * CH) : 0;
            ds[q] = t < nitems ? __ldg(dst + r) - dbase + 2 * (t - r * CH) : 0;
        }
#pragma unroll
        for (int q = 0; q < IU; ++q)
            if (t0 + q * PT < nitems) cp_async16(prod + ds[q], x + cl[q]);
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    // (16 items per thread in one pass -- descriptors, coefficients and copies
    // all in flight together -- was measured slower: 37k vs 16k cycles per batch)
    for (int t0 = threadIdx.x; t0 < nitems; t0 += PT * IU) {
        int ds[IU];
        double cf[IU];
#pragma unroll
        for (int q = 0; q < IU; ++q) {
            const int t = t0 + q * PT, r = t / CH;
            cf[q] = t < nitems ? __ldg(coefs + r) : 0.0;
            ds[q] = t < nitems ? __ldg(dst + r) - dbase + 2 * (t - r * CH) : 0;
        }
#pragma unroll
        for (int q = 0; q < IU; ++q) {
            if (t0 + q * PT >= nitems) break;
            double2 *pp = reinterpret_cast<double2 *>(prod + ds[q]);
            const double2 v = *pp;
            *pp = make_double2(__dmul_rn(cf[q], v.x), __dmul_rn(cf[q], v.y));
        }
    }
}

// sums (and reciprocals) of units [ua, ub) of one direction: batches of whole
// units whose products fit `cap` doubles; a unit larger than `cap` is summed
// straight from its run list by one thread.  Results go to shared memory
// (s_sum / s_rcp, indexed u - ua) for the CTA's own cell pass and to global
// memory (the TV / pricing kernels read the final sums).
__device__ __noinline__ void cl_unit_sums(const int32_t *__restrict__ cells,
                                          const double *__restrict__ coefs,
                                          const int32_t *__restrict__ dst,
                                          const int32_t *__restrict__ ptr, int ua, int ub, int K1,
                                          int kappa, const double *x, double *prod,
                                          double *out_sum, double *s_sum, double *s_rcp, int cap) {
    const int per = K1 * kappa;
    int u0 = ua;
    while (u0 < ub) {
        const int a0 = ptr[u0];
        // a batch [u0, u1) needs its products plus CL_SKEW doubles per unit
        int lo = u0 + 1, hi = ub;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int64_t)(ptr[mid] - a0) * per + CL_SKEW * (mid - u0) <= cap) lo = mid;
            else hi = mid - 1;
        }
        const int u1 = lo;
        if ((int64_t)(ptr[u1] - a0) * per + CL_SKEW * (u1 - u0) <= cap) {
            const int nruns = (ptr[u1] - a0) * K1;
            const int32_t *bc = cells + (int64_t)a0 * K1;
            const double *bf = coefs + (int64_t)a0 * K1;
            const int32_t *bd = dst + (int64_t)a0 * K1;
            const int dbase = a0 * per + CL_SKEW * u0;
            CL_TRACE(0);
            switch (kappa) {
                case 2: cl_products<2>(bc, bf, bd, dbase, nruns, x, prod); break;
                case 4: cl_products<4>(bc, bf, bd, dbase, nruns, x, prod); break;
                default: cl_products<8>(bc, bf, bd, dbase, nruns, x, prod); break;
            }
            CL_TRACE(1);
            __syncthreads();
            CL_TRACE(2);
            for (int u = u0 + (int)threadIdx.x; u < u1; u += PT) {
                const int plo = (ptr[u] - a0) * per + CL_SKEW * (u - u0);
                const double v = chain_sum(prod + plo, (ptr[u + 1] - ptr[u]) * per, true);
                out_sum[u] = v;
                s_sum[u - ua] = v;
                s_rcp[u - ua] = v > 0.0 ? __drcp_rn(v) : 0.0;
            }
            CL_TRACE(3);
            __syncthreads();
            CL_TRACE(4);
        } else {
            if (threadIdx.x == 0) {
                const int rlo = ptr[u0] * K1, rhi = ptr[u0 + 1] * K1;
                const double v = run_list_sum_any(cells + rlo, coefs + rlo, rhi - rlo, x, kappa, 0);
                out_sum[u0] = v;
                s_sum[u0 - ua] = v;
                s_rcp[u0 - ua] = v > 0.0 ? __drcp_rn(v) : 0.0;
            }
            __syncthreads();
        }
        u0 = u1;
    }
}

// Cell passes of ipf_kernel over the blocks [ua, ub) this CTA just summed: an
// item is one fine row (KAP cells along axis 0) of one block, its sum and
// reciprocal come from shared memory, so every load of an item is independent
// (no block-map gather) and no cluster barrier separates sums from cells.
struct ClGeom {
    int nd, lk;                 // dimensions, log2(kappa)
    int fs[GDT_MAX_DIM];        // fine strides
    int cn[GDT_MAX_DIM];        // coarse extents
};

__device__ __forceinline__ int cl_block_origin(int k, const ClGeom &g) {
    int off = 0;
#pragma unroll
    for (int a = 0; a < GDT_MAX_DIM; ++a) {
        if (a >= g.nd) break;
        const int ka = k % g.cn[a];
        k /= g.cn[a];
        off += (ka << g.lk) * g.fs[a];
    }
    return off;
}

// fine offset of row r (digits s_1 .. s_{d-1} in base kappa) inside a block
__device__ __forceinline__ int cl_row_offset(int r, const ClGeom &g) {
    int off = 0;
#pragma unroll
    for (int a = 1; a < GDT_MAX_DIM; ++a) {
        if (a >= g.nd) break;
        off += (r & ((1 << g.lk) - 1)) * g.fs[a];
        r >>= g.lk;
    }
    return off;
}


template <int KAP, bool ROW>
__device__ __forceinline__ void cl_cells(const double *__restrict__ mass, int ua, int ub, int K1,
                                         int lk1, const ClGeom &g, const int *org, bool init,
                                         const double *cur, double *nxt, Red &r_io,
                                         const double *s_sum, const double *s_rcp) {
    // (a local copy: the stores to `nxt` could alias a record reached by reference,
    // which would force its fields through memory on every cell)
    constexpr int CL_IU = KAP <= 4 ? 2 : 1;  // items per thread in flight
    Red r = r_io;
    const int nitems = (ub - ua) * K1;
    for (int it0 = threadIdx.x; it0 < nitems; it0 += PT * CL_IU) {
        double ms[CL_IU][KAP], cv[CL_IU][KAP], sm[CL_IU], rc[CL_IU];
        int st[CL_IU];
#pragma unroll
        for (int q = 0; q < CL_IU; ++q) {
            const int item = it0 + q * PT;
            const bool in = item < nitems;
            const int lu = in ? item >> lk1 : 0, row = item & (K1 - 1);
            st[q] = org[lu] + cl_row_offset(row, g);
            sm[q] = s_sum[lu];
            rc[q] = s_rcp[lu];
#pragma unroll
            for (int i = 0; i < KAP; i += 2) {
                const double2 t = in ? __ldg(reinterpret_cast<const double2 *>(mass + st[q] + i))
                                     : make_double2(0.0, 0.0);
                ms[q][i] = t.x;
                ms[q][i + 1] = t.y;
                if (ROW) {
                    const double2 c2 = (in && !init)
                                           ? *reinterpret_cast<const double2 *>(cur + st[q] + i)
                                           : make_double2(0.0, 0.0);
                    cv[q][i] = c2.x;
                    cv[q][i + 1] = c2.y;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CL_IU; ++q) {
            if (it0 + q * PT >= nitems) break;
            const double acc = sm[q];
            double res[KAP];
#pragma unroll
            for (int i = 0; i < KAP; ++i) {
                const double mi = ms[q][i];
                if (ROW) {
                    if (!init) {
                        const double ai = cv[q][i];
                        range_acc(ai, r.amin, r.amax, r.nonfinite);
                        if (mi > 0.0) r.gap += fabs(__dsub_rn(__dmul_rn(ai, acc), mi));
                    }
                    double an = 0.0;
                    if (mi > 0.0) {
                        if (acc <= 0.0) r.zrow = 1;
                        else an = div_shared(mi, acc, rc[q]);
                    }
                    res[i] = an;
                } else {
                    double bj = 0.0;
                    if (mi > 0.0) {
                        if (acc <= 0.0) r.zcol = 1;
                        else bj = div_shared(mi, acc, rc[q]);
                        range_acc(bj, r.bmin, r.bmax, r.nonfinite);
                        r.gap += fabs(__dsub_rn(mi, __dmul_rn(bj, acc)));
                    }
                    res[i] = bj;
                }
            }
#pragma unroll
            for (int i = 0; i < KAP; i += 2)
                *reinterpret_cast<double2 *>(nxt + st[q] + i) = make_double2(res[i], res[i + 1]);
        }
    }
    r_io = r;
}

template <bool ROW>
__device__ __forceinline__ void cl_cells_any(int kappa, const double *mass, int ua, int ub, int K1,
                                          int lk1, const ClGeom &g, int *org, bool init,
                                          const double *cur, double *nxt, Red &r,
                                          const double *s_sum, const double *s_rcp) {
    for (int u = ua + (int)threadIdx.x; u < ub; u += PT) org[u - ua] = cl_block_origin(u, g);
    __syncthreads();
    switch (kappa) {
        case 2: cl_cells<2, ROW>(mass, ua, ub, K1, lk1, g, org, init, cur, nxt, r, s_sum, s_rcp); break;
        case 4: cl_cells<4, ROW>(mass, ua, ub, K1, lk1, g, org, init, cur, nxt, r, s_sum, s_rcp); break;
        default: cl_cells<8, ROW>(mass, ua, ub, K1, lk1, g, org, init, cur, nxt, r, s_sum, s_rcp); break;
    }
}

// CTA reduction, then the cluster's records combined in rank order (includes
// one cluster barrier; every CTA ends with the same record)
__device__ void cl_reduce_red(Red &r, double *sh, double *xch, unsigned rank, unsigned cs) {
    block_reduce_red(r, sh);
    if (threadIdx.x == 0) {
        double *o = xch + rank * 8;
        o[0] = r.gap;
        o[1] = r.amin;
        o[2] = r.amax;
        o[3] = r.bmin;
        o[4] = r.bmax;
        o[5] = (double)(r.zrow | (r.zcol << 1) | (r.nonfinite << 2));
    }
    cluster_sync_all();
    if (threadIdx.x < cs * 8) sh[threadIdx.x] = ld_gl(xch + threadIdx.x);
    __syncthreads();
    Red o = red_init();
    for (unsigned q = 0; q < cs; ++q) {
        const double *s = sh + q * 8;
        o.gap += s[0];
        o.amin = fmin(o.amin, s[1]);
        o.amax = fmax(o.amax, s[2]);
        o.bmin = fmin(o.bmin, s[3]);
        o.bmax = fmax(o.bmax, s[4]);
        const int fl = (int)s[5];
        o.zrow |= fl & 1;
        o.zcol |= (fl >> 1) & 1;
        o.nonfinite |= (fl >> 2) & 1;
    }
    __syncthreads();
    r = o;
}

constexpr int CL_MAX = 8;       // largest cluster
constexpr int CL_MIN_UNITS = 128;  // the 4th per-pair block of U doubles holds the exchange area

__global__ void __launch_bounds__(PT) ipf_cluster_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu,
    const int64_t *__restrict__ arc_off, const int32_t *__restrict__ row_ptr,
    const int32_t *__restrict__ col_ptr, const double *__restrict__ xi_in, int64_t max_iter,
    G32 f, G32 c, int kappa, int K1, double *__restrict__ out, int32_t *__restrict__ status,
    double *scratch, int64_t stride_pair, const int32_t *__restrict__ rl_cells,
    const double *__restrict__ rl_coef, const int32_t *__restrict__ cl_cells_,
    const double *__restrict__ cl_coef, const int32_t *__restrict__ rl_dst,
    const int32_t *__restrict__ cl_dst, int cap) {
    extern __shared__ double prod[];  // [cap] products | CSR/CSC pointers | sums, reciprocals, origins
    __shared__ double sh[(PT / 32 + 1) * 6 > CL_MAX * 8 ? (PT / 32 + 1) * 6 : CL_MAX * 8];
    __shared__ int part[4];
    const unsigned cs = cluster_size(), rank = cluster_rank_id();
    const int64_t b = blockIdx.x / cs;
    const int N = f.cells, U = c.cells;
    const double *mub = mu + b * N, *nub = nu + b * N;
    const int64_t a0 = arc_off[b];
    const int32_t *rptr = row_ptr + b * (U + 1), *cptr = col_ptr + b * (U + 1);
    const int32_t *rrc = rl_cells + a0 * K1, *crc = cl_cells_ + a0 * K1;
    const double *rrf = rl_coef + a0 * K1, *crf = cl_coef + a0 * K1;
    const int32_t *rrd = rl_dst + a0 * K1, *crd = cl_dst + a0 * K1;
    double *ws = scratch + b * stride_pair;
    double *aA = ws, *aB = ws + N, *bv = ws + 2 * (int64_t)N;
    double *kb = ws + 3 * (int64_t)N, *kta = kb + U, *xch = kta + 2 * (int64_t)U;
    // xch: [0, 64) reduction records, [64, 72) zero-column flags, [80, 88) support counts
    ClGeom g;
    g.nd = f.nd;
    g.lk = kappa == 2 ? 1 : (kappa == 4 ? 2 : 3);
#pragma unroll
    for (int a = 0; a < GDT_MAX_DIM; ++a) {
        g.fs[a] = f.stride[a];
        g.cn[a] = c.n[a];
    }
    const int lk1 = g.lk * (f.nd - 1);  // K1 = 1 << lk1

    // unit ranges balanced by arc count: rank r takes the units whose first
    // arc lies in [A r / cs, A (r + 1) / cs)
    if (threadIdx.x < 4) {
        const int32_t *ptr = threadIdx.x < 2 ? rptr : cptr;
        const unsigned edge = rank + (threadIdx.x & 1);
        int res;
        if (edge == 0) res = 0;
        else if (edge == cs) res = U;
        else {
            const int64_t target = (int64_t)ptr[U] * edge / cs;
            int lo = 0, hi = U;  // first u with ptr[u] >= target
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (ptr[mid] >= target) hi = mid;
                else lo = mid + 1;
            }
            res = lo;
        }
        part[threadIdx.x] = res;
    }
    const int cper = ((N + (int)cs - 1) / (int)cs + 7) & ~7;
    const int c0 = min(N, (int)rank * cper), c1 = min(N, c0 + cper);
    // the pair's CSR / CSC pointers in shared memory (after the products): the
    // batch searches of cl_unit_sums stay on chip; then this CTA's unit sums,
    // their reciprocals and block origins
    int32_t *sp = reinterpret_cast<int32_t *>(prod + cap);
    for (int i = threadIdx.x; i <= U; i += PT) {
        sp[i] = rptr[i];
        sp[U + 1 + i] = cptr[i];
    }
    rptr = sp;
    cptr = sp + U + 1;
    double *s_sum = prod + cap + (U + 2);  // 2 (U + 1) ints = U + 1 doubles, rounded up
    double *s_rcp = s_sum + U;
    int *org = reinterpret_cast<int *>(s_rcp + U);

    // supports, b = ones over the target support, the default xi (quantized.py:317-320)
    double cnt = 0.0;
    for (int i0 = c0 + (int)threadIdx.x; i0 < c1; i0 += PT * 4) {
        double mi[4], ni[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * PT;
            mi[q] = i < c1 ? __ldg(mub + i) : 0.0;
            ni[q] = i < c1 ? __ldg(nub + i) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * PT;
            if (i >= c1) break;
            cnt += (mi[q] > 0.0 ? 1.0 : 0.0) + (ni[q] > 0.0 ? 1.0 : 0.0);
            bv[i] = ni[q] > 0.0 ? 1.0 : 0.0;
        }
    }
    cnt = block_sum<PT>(cnt, sh);
    if (threadIdx.x == 0) xch[80 + rank] = cnt;
    cluster_sync_all();
    cnt = 0.0;
    for (unsigned q = 0; q < cs; ++q) cnt += ld_gl(xch + 80 + q);  // integers: exact in any order
    const double xi = xi_in[b] < 0.0 ? 1e-9 * cnt : xi_in[b];
    const int ru0 = part[0], ru1 = part[1], cu0 = part[2], cu1 = part[3];

    Red r = red_init();
    double *a_cur = aA, *a_nxt = aB;
    cl_unit_sums(rrc, rrf, rrd, rptr, ru0, ru1, K1, kappa, bv, prod, kb, s_sum, s_rcp, cap);
    cl_cells_any<true>(kappa, mub, ru0, ru1, K1, lk1, g, org, true, nullptr, a_cur, r, s_sum, s_rcp);
    cl_reduce_red(r, sh, xch, rank, cs);
    int st = r.zrow ? GDT_PAIR_ZERO_DENOM_ROW : GDT_PAIR_OK;
    int64_t it = 0;
    double gap = INFINITY;
    bool converged = false;
    while (st == GDT_PAIR_OK && it < max_iter) {
        ++it;
        EX_TRACE(0);
#ifdef GDT_IPF_TRACE
        if (blockIdx.x == 0 && threadIdx.x == 0) g_cl_on = it == 10 ? 1 : 0;
#endif
        Red rc = red_init();
        cl_unit_sums(crc, crf, crd, cptr, cu0, cu1, K1, kappa, a_cur, prod, kta, s_sum, s_rcp, cap);
        EX_TRACE(1);
#ifdef GDT_IPF_TRACE
        if (blockIdx.x == 0 && threadIdx.x == 0) g_cl_on = 0;
#endif
        cl_cells_any<false>(kappa, nub, cu0, cu1, K1, lk1, g, org, false, nullptr, bv, rc, s_sum, s_rcp);
        EX_TRACE(2);
        const int zc = __syncthreads_or(rc.zcol);
        if (threadIdx.x == 0) xch[64 + rank] = (double)zc;
        cluster_sync_all();  // C: b complete, flags visible
        EX_TRACE(3);
        {
            int any = 0;
            for (unsigned q = 0; q < cs; ++q) any |= ld_gl(xch + 64 + q) != 0.0;
            if (any) {  // before anything reads b
                st = GDT_PAIR_ZERO_DENOM_COL;
                break;
            }
        }
        cl_unit_sums(rrc, rrf, rrd, rptr, ru0, ru1, K1, kappa, bv, prod, kb, s_sum, s_rcp, cap);
        EX_TRACE(4);
        cl_cells_any<true>(kappa, mub, ru0, ru1, K1, lk1, g, org, false, a_cur, a_nxt, rc, s_sum, s_rcp);
        EX_TRACE(5);
        cl_reduce_red(rc, sh, xch, rank, cs);  // A: next a complete, records folded
        EX_TRACE(6);
        const bool bad_a = rc.amin <= rc.amax &&
                           (rc.amin < 1e-100 || rc.amax > 1e100 || !isfinite(rc.amax));
        const bool bad_b = rc.bmin <= rc.bmax &&
                           (rc.bmin < 1e-100 || rc.bmax > 1e100 || !isfinite(rc.bmax));
        if (bad_a || bad_b || rc.nonfinite) {
            st = GDT_PAIR_OVERFLOW;
            break;
        }
        gap = rc.gap;
        if (gap < xi) {
            converged = true;
            break;
        }
        if (it >= max_iter) break;
        if (rc.zrow) {
            st = GDT_PAIR_ZERO_DENOM_ROW;
            break;
        }
        double *tmp = a_cur;
        a_cur = a_nxt;
        a_nxt = tmp;
    }
    if (rank == 0 && threadIdx.x == 0) {
        status[b] = st;
        double *o = out + b * 8;
        o[0] = 0.0;
        o[1] = 0.0;
        o[2] = 0.0;
        o[3] = gap;
        o[4] = (double)it;
        o[5] = converged ? 1.0 : 0.0;
        o[6] = cnt;
        o[7] = a_cur == aA ? 0.0 : 1.0;
    }
}

// ---------------------------------------------------------------------------
// generic CSR IPF (explicit kernels, ring fallback) -- one CTA
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PT) csr_ipf_kernel(
    const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
    const double *__restrict__ data, const int64_t *__restrict__ tindptr,
    const int32_t *__restrict__ tindices, const double *__restrict__ tdata,
    const double *__restrict__ mu, const double *__restrict__ nu, int64_t nr, int64_t nc,
    double xi, int64_t max_iter, double *__restrict__ a, double *__restrict__ b,
    double *__restrict__ kb, double *__restrict__ kta, double *__restrict__ info,
    int32_t *__restrict__ status) {
    __shared__ double sh[(PT / 32 + 1) * 6];
    for (int64_t j = threadIdx.x; j < nc; j += PT) b[j] = 1.0;
    __syncthreads();
    auto rowpass = [&]() {
        for (int64_t i = threadIdx.x; i < nr; i += PT) {
            double s = 0.0;
            for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e)
                s = __dadd_rn(s, __dmul_rn(data[e], b[indices[e]]));
            kb[i] = s;
        }
    };
    rowpass();
    __syncthreads();
    int st = GDT_PAIR_OK;
    int64_t it = 0;
    double gap = INFINITY;
    bool conv = false;
    while (it < max_iter) {
        ++it;
        Red r = red_init();
        for (int64_t i = threadIdx.x; i < nr; i += PT) {
            if (kb[i] <= 0.0 && mu[i] > 0.0) r.zrow = 1;
            a[i] = kb[i] > 0.0 ? __ddiv_rn(mu[i], kb[i]) : 0.0;
        }
        if (__syncthreads_or(r.zrow)) {
            st = GDT_PAIR_ZERO_DENOM_ROW;
            break;
        }
        for (int64_t j = threadIdx.x; j < nc; j += PT) {
            double s = 0.0;
            for (int64_t e = tindptr[j]; e < tindptr[j + 1]; ++e)
                s = __dadd_rn(s, __dmul_rn(tdata[e], a[tindices[e]]));
            kta[j] = s;
            if (s <= 0.0 && nu[j] > 0.0) r.zcol = 1;
            b[j] = s > 0.0 ? __ddiv_rn(nu[j], s) : 0.0;
        }
        if (__syncthreads_or(r.zcol)) {
            st = GDT_PAIR_ZERO_DENOM_COL;
            break;
        }
        rowpass();
        __syncthreads();
        for (int64_t i = threadIdx.x; i < nr; i += PT) {
            range_acc(a[i], r.amin, r.amax, r.nonfinite);
            r.gap += fabs(__dsub_rn(__dmul_rn(a[i], kb[i]), mu[i]));
        }
        for (int64_t j = threadIdx.x; j < nc; j += PT) {
            range_acc(b[j], r.bmin, r.bmax, r.nonfinite);
            r.gap += fabs(__dsub_rn(nu[j], __dmul_rn(b[j], kta[j])));
        }
        block_reduce_red(r, sh);
        const bool bad_a =
            r.amin <= r.amax && (r.amin < 1e-100 || r.amax > 1e100 || !isfinite(r.amax));
        const bool bad_b =
            r.bmin <= r.bmax && (r.bmin < 1e-100 || r.bmax > 1e100 || !isfinite(r.bmax));
        if (bad_a || bad_b || r.nonfinite) {
            st = GDT_PAIR_OVERFLOW;
            break;
        }
        gap = r.gap;
        if (gap < xi) {
            conv = true;
            break;
        }
    }
    if (threadIdx.x == 0) {
        info[0] = (double)it;
        info[1] = gap;
        info[2] = conv ? 1.0 : 0.0;
        info[3] = 0.0;
        status[0] = st;
    }
}

__device__ __forceinline__ double grid_cost64(int64_t i, int64_t j, const Grid &f, double p,
                                              const double *table) {
    int64_t sq = 0;
    for (int a = f.nd - 1; a >= 0; --a) {
        const int64_t xi = i / f.stride[a], xj = j / f.stride[a];
        i -= xi * f.stride[a];
        j -= xj * f.stride[a];
        sq += (xi - xj) * (xi - xj);
    }
    return cost_from_sq(sq, p, table);
}

__global__ void price_coo_kernel(const int64_t *__restrict__ row, const int64_t *__restrict__ col,
                                 const double *__restrict__ mass, int64_t nnz,
                                 const double *__restrict__ a, const double *__restrict__ b,
                                 const double *__restrict__ table, double p, Grid f,
                                 double *__restrict__ part) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double fitted = __dmul_rn(__dmul_rn(a[row[e]], mass[e]), b[col[e]]);
        acc += fitted * grid_cost64(row[e], col[e], f, p, table);
    }
    acc = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void sum_parts_kernel(const double *__restrict__ part, int count, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < count; ++i) s += part[i];
        out[0] = s;
    }
}

// ---------------------------------------------------------------------------
// Coarse-level primal stage (fp32 mode, uniform kernel, C-bar supplied).
//
// With W_ts = W for every cell pair of an arc, every scaling is a per-block
// quotient of the masses (a_t = mu_t / KB_k, b_s = nu_s / KTA_l), so the
// sweep of sinkhorn.py:124-141 closes on the coarse plan:
//   KTA_l = sum_{k -> l} m_kl W S_k,   S_k = sum_{t in X_k} a_t = mu~_k / KB_k,
//   KB_k  = sum_{l <- k} m_kl W B_l,   B_l = sum_{s in Y_l} b_s = nu~_l / KTA_l,
// b = 1 on the target support at the start (B_l = its count).  A sweep costs
// O(arcs) instead of O(cells); the reference's checks keep their order: zero
// row (top of a sweep), zero column, scale range of a then b (from each
// block's extreme positive masses: correctly rounded division by a positive
// constant is monotone), then the gap -- here the coarse residual
// |S_k KB'_k - mu~_k| + |nu~_l - B_l KTA_l| (the fine one up to rounding).
// Pricing needs no fine pass:
//   sum_{t in X_k, s in Y_l} a_t b_s C_ts = G_kl / (KB_k KTA_l) = C-bar_kl S_k B_l
// with G_kl = sum mu_t nu_s C_ts the numerator of C-bar (costs.py:128-171),
// which the weighted-cost bound computes anyway: transport^p is the fitted
// coarse plan priced by C-bar.  The block statistics come from the SumPool
// pass (gdt_sumpool_stats_f64); the only fine pass left is the weighted TV of
// the fitted marginals, cell by cell with the reference's arithmetic
// (tv_pass_kernel, grid-wide).  Summation orders differ from scipy's (the
// fp32-mode contract is 1e-5 on the bounds); C-bar for p != 2 carries the
// fp32 kernel's rounding (<= 3.8e-6 relative per entry), for p = 2 it comes
// from fp64 block moments (~1e-14).
//
// primal_coarse_kernel: one CTA per pair, the plan in shared memory.  Block
// sums over arcs run one thread per block, except blocks with more than
// CB_HEAVY arcs (skewed plans): those are summed by a warp (lane-strided,
// fixed butterfly: deterministic) so no thread serialises a long arc list.
// ---------------------------------------------------------------------------
constexpr int CT = 512;       // threads of primal_coarse_kernel
constexpr int CB_HEAVY = 8;  // arcs above which a block's sum goes to a warp
enum { CB_MLO, CB_MHI, CB_NLO, CB_NHI, CB_CMU, CB_CNU, CB_S, CB_B, CB_K0, CB_K1, CB_KTA, CB_RK,
       CB_S1, CB_NF };

struct CoarsePlan {
    int rp, cp, rcol, rcoef, crow, ccoef, arow, heavy, perm, blk, total;
};

__host__ __device__ inline CoarsePlan coarse_plan(int n) {
    CoarsePlan m;
    const int cap = 2 * n;
    int o = 0;
    m.rp = o;
    o = fp_al(o + 4 * (n + 1));
    m.cp = o;
    o = fp_al(o + 4 * (n + 1));
    m.rcol = o;
    o = fp_al(o + 4 * cap);
    m.rcoef = o;
    o = fp_al(o + 8 * cap);
    m.crow = o;
    o = fp_al(o + 4 * cap);
    m.ccoef = o;
    o = fp_al(o + 8 * cap);
    m.arow = o;
    o = fp_al(o + 4 * cap);
    m.heavy = o;  // heavy row blocks, then heavy column blocks
    o = fp_al(o + 4 * 2 * n);
    m.perm = o;  // light row blocks, then light column blocks, by descending degree
    o = fp_al(o + 4 * 2 * n);
    m.blk = o;
    o = fp_al(o + 8 * CB_NF * n);
    m.total = o;
    return m;
}

struct CoarseRed {
    double gap, alo, ahi, blo, bhi;
    int flags;  // 1 zero row (next sweep), 2 zero column, 4 non-finite
};

__device__ __forceinline__ CoarseRed cr_init() {
    return CoarseRed{0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0};
}

// deterministic CTA reduction: xor butterflies per warp, then warp 0 folds
// the per-warp records in warp order; every thread gets the result
__device__ CoarseRed cr_reduce(CoarseRed r, CoarseRed *sh) {
    auto fold = [](CoarseRed &x) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            x.gap += __shfl_xor_sync(0xffffffffu, x.gap, o);
            x.alo = fmin(x.alo, __shfl_xor_sync(0xffffffffu, x.alo, o));
            x.ahi = fmax(x.ahi, __shfl_xor_sync(0xffffffffu, x.ahi, o));
            x.blo = fmin(x.blo, __shfl_xor_sync(0xffffffffu, x.blo, o));
            x.bhi = fmax(x.bhi, __shfl_xor_sync(0xffffffffu, x.bhi, o));
            x.flags |= __shfl_xor_sync(0xffffffffu, x.flags, o);
        }
    };
    fold(r);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = r;
    __syncthreads();
    if (w == 0) {
        CoarseRed o = lane < CT / 32 ? sh[lane] : cr_init();
        fold(o);
        if (lane == 0) sh[CT / 32] = o;
    }
    __syncthreads();
    const CoarseRed out = sh[CT / 32];
    __syncthreads();
    return out;
}

__device__ __forceinline__ double cr_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        double x = lane < CT / 32 ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) sh[CT / 32] = x;
    }
    __syncthreads();
    const double out = sh[CT / 32];
    __syncthreads();
    return out;
}

// out[u] = sum_{e in [ptr[u], ptr[u+1])} coef[e] * x[idx[e]] for every block u:
// light blocks one thread each, visited in descending degree (`perm`, so the
// lanes of a warp run near-equal trip counts), heavy ones (listed in `heavy`)
// one warp each.  Each block's sum runs in its own fixed arc order.
__device__ __forceinline__ void coarse_matvec(const int *ptr, const int *idx, const double *coef,
                                              const double *x, double *out, const int *perm,
                                              int nlight, const int *heavy, int nheavy) {
    for (int j = threadIdx.x; j < nlight; j += CT) {
        const int u = perm[j];
        const int e0 = ptr[u], e1 = ptr[u + 1];
        double s = 0.0;
        for (int e = e0; e < e1; ++e) s += coef[e] * x[idx[e]];
        out[u] = s;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int h = w; h < nheavy; h += CT / 32) {
        const int u = heavy[h], e0 = ptr[u], e1 = ptr[u + 1];
        double s = 0.0;
        for (int e = e0 + lane; e < e1; e += 32) s += coef[e] * x[idx[e]];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[u] = s;
    }
}

// Smallest / largest scaling of a block (extreme masses over one denominator)
// folded into the running range.  The range is only ever compared with 1e-100
// and 1e100 (_check_scale_range, sinkhorn.py:137-138), so the quotients come
// from one multiplication by the correctly rounded reciprocal (relative error
// < 2^-51) unless that lands within 1e-7 of a threshold or is not a positive
// finite number -- then the correctly rounded divisions decide, as before.
__device__ __forceinline__ void coarse_range(double mlo, double mhi, double den, double rk,
                                             double &rlo, double &rhi, int &flags) {
    double lo = __dmul_rn(mlo, rk), hi = __dmul_rn(mhi, rk);
    if (!(lo > 1.0000001e-100 && hi < 0.9999999e100)) {
        lo = div_shared(mlo, den, rk);
        hi = div_shared(mhi, den, rk);
    }
    if (isnan(lo) || isnan(hi) || !isfinite(hi)) flags |= 4;
    if (lo > 0.0) rlo = fmin(rlo, lo);
    if (hi > 0.0) rhi = fmax(rhi, hi);
}

__global__ void __launch_bounds__(CT, 1) primal_coarse_kernel(
    const double *__restrict__ mu_c, const double *__restrict__ nu_c,
    const double *__restrict__ stats, const double *__restrict__ cbar,
    const int64_t *__restrict__ arc_off, const int32_t *__restrict__ row_ptr,
    const int32_t *__restrict__ row_arc_col, const double *__restrict__ row_arc_mass,
    const int32_t *__restrict__ col_ptr, const int32_t *__restrict__ col_arc_row,
    const double *__restrict__ col_arc_mass, const double *__restrict__ W,
    const double *__restrict__ xi_in, int64_t max_iter, int n, int64_t batch,
    double *__restrict__ blk_out, double *__restrict__ out, int32_t *__restrict__ status) {
    __shared__ CoarseRed shr[CT / 32 + 1];
    __shared__ double shd[CT / 32 + 1];
    __shared__ int nheavy_s[2];
    __shared__ int dcnt[2][CB_HEAVY + 2];
    extern __shared__ __align__(16) unsigned char csm[];
    const int64_t b = blockIdx.x;
    const double Wu = W[0];
    const double *mcb = mu_c + b * n, *ncb = nu_c + b * n;
    const double *smu = stats + b * n * 3, *snu = stats + (batch + b) * n * 3;
    const int64_t a0 = arc_off[b];
    const int A = (int)(arc_off[b + 1] - a0);
    const CoarsePlan L = coarse_plan(n);
    int *rp = reinterpret_cast<int *>(csm + L.rp), *cp = reinterpret_cast<int *>(csm + L.cp);
    int *rcol = reinterpret_cast<int *>(csm + L.rcol), *crow = reinterpret_cast<int *>(csm + L.crow);
    int *arow = reinterpret_cast<int *>(csm + L.arow);
    int *hrow = reinterpret_cast<int *>(csm + L.heavy), *hcol = hrow + n;
    int *prow = reinterpret_cast<int *>(csm + L.perm), *pcol = prow + n;
    double *rcoef = reinterpret_cast<double *>(csm + L.rcoef);
    double *ccoef = reinterpret_cast<double *>(csm + L.ccoef);
    double *blk = reinterpret_cast<double *>(csm + L.blk);
    double *Bmlo = blk + CB_MLO * n, *Bmhi = blk + CB_MHI * n, *Bnlo = blk + CB_NLO * n,
           *Bnhi = blk + CB_NHI * n, *Bcmu = blk + CB_CMU * n, *Bcnu = blk + CB_CNU * n,
           *BB = blk + CB_B * n, *KTA = blk + CB_KTA * n;
    // S_k of the current sweep and, written by the row pass, of the next; 1 / kb
    // is read and replaced by the same thread of the row pass (no second buffer)
    double *BS = blk + CB_S * n, *RK = blk + CB_RK * n;
    double *BSn = blk + CB_S1 * n;
    double *Kcur = blk + CB_K0 * n, *Knext = blk + CB_K1 * n;

    // ---- the pair's coarse plan and block statistics into shared memory
    if (threadIdx.x < 2) nheavy_s[threadIdx.x] = 0;
    if (threadIdx.x < 2 * (CB_HEAVY + 2)) (&dcnt[0][0])[threadIdx.x] = 0;
    for (int i = threadIdx.x; i <= n; i += CT) {
        rp[i] = row_ptr[b * (n + 1) + i];
        cp[i] = col_ptr[b * (n + 1) + i];
    }
    for (int e = threadIdx.x; e < A; e += CT) {
        rcol[e] = row_arc_col[a0 + e];
        rcoef[e] = __dmul_rn(row_arc_mass[a0 + e], Wu);
        crow[e] = col_arc_row[a0 + e];
        ccoef[e] = __dmul_rn(col_arc_mass[a0 + e], Wu);
    }
    double cnt = 0.0;
    for (int k = threadIdx.x; k < n; k += CT) {
        Bmlo[k] = smu[3 * k];
        Bmhi[k] = smu[3 * k + 1];
        Bcmu[k] = smu[3 * k + 2];
        Bnlo[k] = snu[3 * k];
        Bnhi[k] = snu[3 * k + 1];
        Bcnu[k] = snu[3 * k + 2];
        cnt += Bcmu[k] + Bcnu[k];
    }
    __syncthreads();
    // heavy blocks (> CB_HEAVY arcs) per side; the light ones bucketed by
    // degree (counting sort, descending) for the thread-per-block sums
    for (int k = threadIdx.x; k < n; k += CT) {
        for (int e = rp[k]; e < rp[k + 1]; ++e) arow[e] = k;
        const int dr = rp[k + 1] - rp[k], dc = cp[k + 1] - cp[k];
        if (dr > CB_HEAVY) hrow[atomicAdd(&nheavy_s[0], 1)] = k;
        else atomicAdd(&dcnt[0][CB_HEAVY - dr], 1);
        if (dc > CB_HEAVY) hcol[atomicAdd(&nheavy_s[1], 1)] = k;
        else atomicAdd(&dcnt[1][CB_HEAVY - dc], 1);
    }
    __syncthreads();
    if (threadIdx.x < 2) {  // exclusive scan of the degree buckets
        int acc = 0;
        for (int q = 0; q <= CB_HEAVY; ++q) {
            const int c = dcnt[threadIdx.x][q];
            dcnt[threadIdx.x][q] = acc;
            acc += c;
        }
        dcnt[threadIdx.x][CB_HEAVY + 1] = acc;  // number of light blocks
    }
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += CT) {
        const int dr = rp[k + 1] - rp[k], dc = cp[k + 1] - cp[k];
        if (dr <= CB_HEAVY) prow[atomicAdd(&dcnt[0][CB_HEAVY - dr], 1)] = k;
        if (dc <= CB_HEAVY) pcol[atomicAdd(&dcnt[1][CB_HEAVY - dc], 1)] = k;
    }
    cnt = cr_sum(cnt, shd);  // (its barriers also publish the tables above)
    const int nhr = nheavy_s[0], nhc = nheavy_s[1];
    const int nlr = n - nhr, nlc = n - nhc;
    // the heavy lists and the buckets are sets: their order only decides which
    // thread or warp sums a block, never the order of a block's own sum
    const double xi = xi_in[b] < 0.0 ? 1e-9 * cnt : xi_in[b];

    // ---- kb = K b with b = 1 on the target support (sinkhorn.py:119-120)
    coarse_matvec(rp, rcol, rcoef, Bcnu, Kcur, prow, nlr, hrow, nhr);
    __syncthreads();
    int zrow = 0;
    for (int k = threadIdx.x; k < n; k += CT)
        if (Bcmu[k] > 0.0 && Kcur[k] <= 0.0) zrow = 1;
    int st = __syncthreads_or(zrow) ? GDT_PAIR_ZERO_DENOM_ROW : GDT_PAIR_OK;
    int64_t it = 0;
    double gap = INFINITY;
    bool converged = false;
    // a = mu / kb: block sums S_k (quotients correctly rounded: div_shared,
    // Markstein from one reciprocal per denominator); later sweeps get theirs
    // from the row pass of the sweep before
    for (int k = threadIdx.x; k < n; k += CT) {
        const double den = Kcur[k];
        const double rk = fp_rcp(den);
        RK[k] = rk;
        BS[k] = (Bcmu[k] > 0.0 && den > 0.0) ? div_shared(mcb[k], den, rk) : 0.0;
    }
    __syncthreads();
    while (st == GDT_PAIR_OK && it < max_iter) {
        ++it;
        EX_TRACE(0);
        EX_TRACE(1);
        // kta = K^T a
        coarse_matvec(cp, crow, ccoef, BS, KTA, pcol, nlc, hcol, nhc);
        __syncthreads();
        EX_TRACE(2);
        // zero-column check, b = nu / kta: block sums B_l, column residual, range(b)
        CoarseRed r = cr_init();
        for (int l = threadIdx.x; l < n; l += CT) {
            const double s = KTA[l];
            double bl = 0.0;
            if (Bcnu[l] > 0.0) {
                if (s <= 0.0) {
                    r.flags |= 2;
                } else {
                    const double rs = __drcp_rn(s);
                    bl = div_shared(ncb[l], s, rs);
                    r.gap += fabs(__dsub_rn(ncb[l], __dmul_rn(bl, s)));
                    coarse_range(Bnlo[l], Bnhi[l], s, rs, r.blo, r.bhi, r.flags);
                }
            }
            BB[l] = bl;
        }
        __syncthreads();
        EX_TRACE(3);
        // kb' = K b
        coarse_matvec(rp, rcol, rcoef, BB, Knext, prow, nlr, hrow, nhr);
        __syncthreads();
        EX_TRACE(4);
        // range of a (from kb), the row residual, the next sweep's zero-row check
        for (int k = threadIdx.x; k < n; k += CT) {
            const double s = Knext[k];
            const double rn = fp_rcp(s);
            double sn = 0.0;
            if (Bcmu[k] > 0.0) {
                const double den = Kcur[k];
                if (den > 0.0) coarse_range(Bmlo[k], Bmhi[k], den, RK[k], r.alo, r.ahi, r.flags);
                r.gap += fabs(__dsub_rn(__dmul_rn(BS[k], s), mcb[k]));
                if (s <= 0.0) r.flags |= 1;
                else sn = div_shared(mcb[k], s, rn);
            }
            RK[k] = rn;  // the next sweep's a = mu / kb'
            BSn[k] = sn;
        }
        EX_TRACE(5);
        const CoarseRed q = cr_reduce(r, shr);
        EX_TRACE(6);
        if (q.flags & 2) {
            st = GDT_PAIR_ZERO_DENOM_COL;
            break;
        }
        if (fp_bad(q.alo, q.ahi) || fp_bad(q.blo, q.bhi) || (q.flags & 4)) {
            st = GDT_PAIR_OVERFLOW;
            break;
        }
        gap = q.gap;
        if (gap < xi) {
            converged = true;
            break;
        }
        if (it >= max_iter) break;
        if (q.flags & 1) {  // the check at the top of the next sweep
            st = GDT_PAIR_ZERO_DENOM_ROW;
            break;
        }
        double *t = Kcur;  // kb' defines a of the next sweep
        Kcur = Knext;
        Knext = t;
        t = BS;
        BS = BSn;
        BSn = t;
    }
    // ---- pricing: the fitted coarse plan S_k (m W) B_l against C-bar (flat
    //      over the arcs: balanced; per-thread partials in a fixed order)
    double price = 0.0;
    const bool ok = st == GDT_PAIR_OK && it >= 1;
    if (ok)
        for (int e = threadIdx.x; e < A; e += CT) {
            const int k = arow[e], l = rcol[e];
            price += __dmul_rn(__dmul_rn(BS[k], rcoef[e]), BB[l]) *
                     __ldg(cbar + ((int64_t)b * n + k) * n + l);
        }
    price = cr_sum(price, shd);
    // per-block denominators of the final a (kb), of the plan's row marginal
    // (kb') and of b (kta), for the weighted-TV pass
    double *bo = blk_out + b * 3 * n;
    for (int k = threadIdx.x; k < n; k += CT) {
        bo[k] = ok ? Kcur[k] : 0.0;
        bo[n + k] = ok ? Knext[k] : 0.0;
        bo[2 * n + k] = ok ? KTA[k] : 0.0;
    }
    if (threadIdx.x == 0) {
        status[b] = st;
        double *o = out + b * 8;
        o[0] = price;
        o[1] = 0.0;
        o[2] = 0.0;
        o[3] = gap;
        o[4] = (double)it;
        o[5] = converged ? 1.0 : 0.0;
        o[6] = cnt;
        o[7] = 0.0;
    }
}

// Weighted TV of the fitted plan's marginals (quantized.py:357-363):
//   mu^ = a (K b) = a KB'_k, nu^ = b (K^T a) = b KTA_l, a = mu / KB_k, b = nu / KTA_l,
// inner sums sum_i w_i |mu^_i - mu_i| and sum_i w_i |nu^_i - nu_i| with the
// reference's per-cell arithmetic (correctly rounded quotients; w = tv_weights
// of the padded grid, measures.py:289-296).  Grid-wide, coalesced; one
// partial pair per CTA (fixed order: deterministic).
constexpr int TVT = 256, TV_CELLS = 8;  // threads, cells per thread of tv_pass_kernel

__global__ void __launch_bounds__(TVT) tv_pass_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu,
    const double *__restrict__ blk, const int32_t *__restrict__ status,
    const double *__restrict__ tv_w, const int32_t *__restrict__ bmap, int N, int n,
    double *__restrict__ part) {
    __shared__ double sh[32];
    const int64_t b = blockIdx.y;
    double tmu = 0.0, tnu = 0.0;
    if (status[b] == GDT_PAIR_OK) {
        const double *mub = mu + b * N, *nub = nu + b * N;
        const double *k0 = blk + b * 3 * n, *k1 = k0 + n, *kt = k0 + 2 * n;
        const int base = blockIdx.x * TVT * TV_CELLS + threadIdx.x;
        // every independent load first (masses, weights, block ids), then the
        // per-block denominators, then the arithmetic
        double mv[TV_CELLS], nv[TV_CELLS], wv[TV_CELLS];
        int kv[TV_CELLS];
#pragma unroll
        for (int q = 0; q < TV_CELLS; ++q) {
            const int i = base + q * TVT;
            const bool in = i < N;
            mv[q] = in ? mub[i] : 0.0;
            nv[q] = in ? nub[i] : 0.0;
            wv[q] = in ? __ldg(tv_w + i) : 0.0;
            kv[q] = in ? __ldg(bmap + i) : 0;
        }
        double d0[TV_CELLS], d1[TV_CELLS], dt[TV_CELLS];
#pragma unroll
        for (int q = 0; q < TV_CELLS; ++q) {
            d0[q] = __ldg(k0 + kv[q]);
            d1[q] = __ldg(k1 + kv[q]);
            dt[q] = __ldg(kt + kv[q]);
        }
#pragma unroll
        for (int q = 0; q < TV_CELLS; ++q) {
            if (mv[q] > 0.0) {
                const double ai = fp_scale(mv[q], d0[q], fp_rcp(d0[q]));
                tmu += wv[q] * fabs(__dsub_rn(__dmul_rn(ai, d1[q]), mv[q]));
            }
            if (nv[q] > 0.0) {
                const double bi = fp_scale(nv[q], dt[q], fp_rcp(dt[q]));
                tnu += wv[q] * fabs(__dsub_rn(__dmul_rn(bi, dt[q]), nv[q]));
            }
        }
    }
    tmu = block_sum<TVT>(tmu, sh);
    tnu = block_sum<TVT>(tnu, sh);
    if (threadIdx.x == 0) {
        double *pp = part + ((int64_t)b * gridDim.x + blockIdx.x) * 2;
        pp[0] = tmu;
        pp[1] = tnu;
    }
}

// scratch layout per pair: [aA N][aB N][b N][kb U][kta U]; then, after all
// pairs: moments [B, n, MW], tv partials [B, tv_ctas, 2], price partials
// [B, pr_ctas]
// lanes per coarse block in moments_tv_kernel: a power of two dividing
// kappa^d with >= 4 cells per lane (the group fold costs shuffles), <= 32
inline int tv_lanes(const Grid &f, const Grid &c) {
    const int64_t m = f.cells / c.cells;
    int lb = 1;
    while (lb < 32 && lb * 8 <= m && m % (lb * 2) == 0) lb *= 2;
    return lb;
}

struct PrimalLayout {
    int64_t stride_pair, mom_off, tv_off, pr_off, pc_off, bm_off, fp_off, ar_off, rl_off, prod_off,
        total,
        tv_ctas, pr_ctas, runs;
};

inline PrimalLayout primal_layout(int64_t batch, const Grid &f, const Grid &c, bool uniform,
                                  bool p2, int64_t max_arcs) {
    PrimalLayout L;
    const int64_t U = uniform ? c.cells : f.cells;
    L.stride_pair = 3 * f.cells + 4 * U;  // aA, aB, b, kb, kta, reciprocals / S, B
    L.mom_off = batch * L.stride_pair;
    const int64_t MW = 2 * (f.nd + 2);
    L.tv_ctas = (c.cells * tv_lanes(f, c) + MT - 1) / MT;
    // brute-force pricing has one item per (arc, row offset): f.cells / c.cells = kappa^d
    const int64_t items = (uniform && p2) ? max_arcs : max_arcs * (f.cells / c.cells);
    L.pr_ctas = (items + MT - 1) / MT;
    L.tv_off = L.mom_off + batch * c.cells * MW;
    L.pr_off = L.tv_off + batch * L.tv_ctas * 2;
    L.pc_off = L.pr_off + batch * L.pr_ctas;       // packed arc coordinates (int64)
    L.bm_off = L.pc_off + 2 * batch * max_arcs;    // fine cell -> coarse block (int32)
    L.fp_off = L.bm_off + (f.cells + 1) / 2;        // ipf_fast_kernel partials
    L.ar_off = L.fp_off + batch * 5 * FCS_MAX * (int64_t)(sizeof(FastPart) / sizeof(double));
    L.rl_off = L.ar_off + (batch * max_arcs + 1) / 2;  // arc -> row block (int32)
    // uniform exact IPF: run lists per direction, coefficients (f64) then cells (int32)
    const int64_t kap = f.n[0] / c.n[0];
    L.runs = uniform ? batch * max_arcs * (f.cells / c.cells / kap) : 0;
    L.prod_off = 0;  // (two-phase products live in shared memory)
    // (+ the product slots of the cluster kernel, int32 per run and direction)
    L.total = L.rl_off + 2 * L.runs + L.runs + L.runs;
    return L;
}

}  // namespace gdt

using namespace gdt;

extern "C" int64_t gdt_primal_scratch_bytes(int64_t batch, int ndim, const int64_t *dims,
                                            int kappa, int kernel_uniform) {
    Grid f, c;
    if (!make_grid(f, ndim, dims) || !make_coarse(c, f, kappa)) return -1;
    // a basic solution has at most 2n - 1 positive arcs (ns + nt - 1)
    // sized for the brute-force pricing layout (the larger one)
    const PrimalLayout L = primal_layout(batch, f, c, kernel_uniform != 0, false, 2 * c.cells);
    return (int64_t)sizeof(double) * L.total;
}

extern "C" int gdt_primal_upscale(const double *mu, const double *nu, const double *mu_c,
                                  const double *nu_c, const double *stats, const double *cbar,
                                  const double *tv_w, const int32_t *bmap_in,
                                  const int64_t *arc_off,
                                  const int32_t *row_ptr, const int32_t *row_arc_col,
                                  const double *row_arc_mass, const int32_t *col_ptr,
                                  const int32_t *col_arc_row, const double *col_arc_mass,
                                  const double *kernel_w, int kernel_uniform, const double *xi,
                                  int64_t max_iter, double p, int64_t batch, int ndim,
                                  const int64_t *dims, int kappa, const double *cost_table,
                                  int64_t max_sq, int mode, double *out, int32_t *status,
                                  void *scratch, void *stream) {
    Grid f, c;
    GDT_CHECK_ARG(make_grid(f, ndim, dims) && make_coarse(c, f, kappa),
                  "gdt_primal_upscale: dims must be positive multiples of kappa");
    GDT_CHECK_ARG(f.cells < (1ll << 31), "gdt_primal_upscale: grid too large for int32 indexing");
    GDT_CHECK_ARG(p >= 1.0 && max_iter >= 1 && batch >= 0, "gdt_primal_upscale: bad p/max_iter");
    int64_t need_sq = 0;
    for (int a = 0; a < ndim; ++a) need_sq += (dims[a] - 1) * (dims[a] - 1);
    GDT_CHECK_ARG(p == 1.0 || p == 2.0 || (cost_table != nullptr && max_sq >= need_sq),
                  "gdt_primal_upscale: cost_table required for p not in {1, 2}");
    if (batch == 0) return GDT_OK;
    cudaStream_t st = as_stream(stream);
    const bool uni = kernel_uniform != 0;
    const PrimalLayout L = primal_layout(batch, f, c, uni, p == 2.0, 2 * c.cells);
    double *ws = (double *)scratch;
    const G32 f32 = to32(f), c32 = to32(c);
    GDT_CHECK_ARG(c.n[0] < 65536 && c.n[1] < 65536 && c.n[2] < 65536 && c.n[3] < 65536,
                  "gdt_primal_upscale: coarse axes must be < 65536");
    const bool fast_ipf = uni && mode == GDT_MODE_FAST;
    if (fast_ipf && cbar != nullptr && mu_c != nullptr && nu_c != nullptr && stats != nullptr &&
        tv_w != nullptr && bmap_in != nullptr) {
        const CoarsePlan plan = coarse_plan((int)c.cells);
        // (<= 190 KB of dynamic shared memory: Nsight Compute reserves part of an SM's
        // shared memory, a 194 KB launch failed under its graph replay)
        if (plan.total <= 190 * 1024) {
            // the whole primal stage at the coarse level: sweeps + pricing
            // (one CTA per pair), the weighted-TV pass (grid-wide), the fold
            const int n = (int)c.cells;
            double *blk = ws;                             // [batch, 3, n]
            double *tvp = ws + batch * 3 * c.cells;       // [batch, tv_ctas, 2]
            const int tv_ctas = (int)((f.cells + TVT * TV_CELLS - 1) / (TVT * TV_CELLS));
            if (plan.total > 48 * 1024)
                cudaFuncSetAttribute(primal_coarse_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, plan.total);
            primal_coarse_kernel<<<(unsigned)batch, CT, plan.total, st>>>(
                mu_c, nu_c, stats, cbar, arc_off, row_ptr, row_arc_col, row_arc_mass, col_ptr,
                col_arc_row, col_arc_mass, kernel_w, xi, max_iter, n, batch, blk, out, status);
            tv_pass_kernel<<<dim3((unsigned)tv_ctas, (unsigned)batch), TVT, 0, st>>>(
                mu, nu, blk, status, tv_w, bmap_in, (int)f.cells, n, tvp);
            finish_kernel<<<grid_size(batch * 32, 128), 128, 0, st>>>(tvp, tv_ctas, nullptr, 0,
                                                                     status, out, batch);
            return cuda_status("gdt_primal_upscale (coarse)");
        }
    }
    int64_t *rpc = reinterpret_cast<int64_t *>(ws + L.pc_off);
    int64_t *cpc = rpc + batch * 2 * c.cells;
    const int64_t per_pair = 2 * c.cells;
    int32_t *bmap = reinterpret_cast<int32_t *>(ws + L.bm_off);
    if (!fast_ipf) {  // packed arc coordinates and the block map of ipf_kernel
        pack_coords_kernel<<<grid_size(batch * per_pair, 256), 256, 0, st>>>(
            row_arc_col, arc_off, per_pair, batch, c32, rpc);
        pack_coords_kernel<<<grid_size(batch * per_pair, 256), 256, 0, st>>>(
            col_arc_row, arc_off, per_pair, batch, c32, cpc);
        if (uni) block_map_kernel<<<grid_size(f.cells, 256), 256, 0, st>>>(f32, c32, kappa, bmap);
    }
    const size_t sxb = sizeof(double) * f.cells;
    const int use_smem = sxb <= 160 * 1024;
    size_t dyn = use_smem ? sxb : 0;
    // exact-order unit sums in two phases (products, then the chains) when the
    // staged vector and one direction's products fit in shared memory
    int prod_smem = 0;
    if (uni) {
        // all of one direction's products when they fit beside the staged
        // vector, else batches of up to 20480 (160 KB)
        const int64_t prods = 2 * c.cells * (f.cells / c.cells);
        const int64_t base = use_smem ? ((f.cells + 1) & ~1ll) : 0;
        const int64_t room = (184 * 1024) / (int64_t)sizeof(double) - base;  // see the 190 KB note above
        const int64_t capd = std::min<int64_t>(prods, std::min<int64_t>(room, 20480));
        if (capd >= std::min<int64_t>(prods, 4096)) {
            prod_smem = (int)(capd & ~1ll);
            dyn = sizeof(double) * (base + prod_smem) + sizeof(int32_t) * 2 * (c.cells + 1);
        }
    }
    if (fast_ipf) {
        // one cluster of ceil(units / FT) <= 8 CTAs per pair; a unit is one
        // fine row of a block for kappa in {2, 4, 8} with kappa^(d-1) <= 32
        int rows = 1;
        for (int a = 1; a < ndim; ++a) rows *= kappa;
        const bool tmpl = (kappa == 2 || kappa == 4 || kappa == 8) && rows <= 32;
        GDT_CHECK_ARG(tmpl || kappa <= 16, "gdt_primal_upscale: fast IPF needs kappa <= 16");
        const int64_t units = c.cells * (tmpl ? rows : 1);
        const unsigned csz = (unsigned)std::min<int64_t>(FCS_MAX, (units + FT - 1) / FT);
        const int64_t upc = ((units + csz - 1) / csz + 31) / 32 * 32;
        const int64_t bpc = upc / (tmpl ? rows : 1);
        // arcs of one CTA's blocks in shared memory up to `cap` per side
        const int cap = (int)std::min<int64_t>(2 * c.cells, 1024);
        const FpSmem plan = fp_smem_plan((int)c.cells, (int)bpc, (int)upc, cap);
        GDT_CHECK_ARG(plan.total <= 200 * 1024, "gdt_primal_upscale: coarse grid too large for the fast IPF");
        const size_t fsmem = (size_t)plan.total;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(batch * csz));
        cfg.blockDim = dim3(FT);
        cfg.dynamicSmemBytes = fsmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csz;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        auto go = [&](auto kern) {
            if (fsmem > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
            return cudaLaunchKernelEx(&cfg, kern, mu, nu, arc_off, row_ptr, row_arc_col,
                                      row_arc_mass, col_ptr, col_arc_row, col_arc_mass, kernel_w,
                                      xi, max_iter, f32, c32, kappa, out, status, ws,
                                      L.stride_pair, cap);
        };
        cudaError_t e;
        if (!tmpl) e = go(ipf_fast_kernel<0>);
        else if (kappa == 2) e = go(ipf_fast_kernel<2>);
        else if (kappa == 4) e = go(ipf_fast_kernel<4>);
        else e = go(ipf_fast_kernel<8>);
        if (e != cudaSuccess) {
            set_error(std::string("gdt_primal_upscale: ipf_fast_kernel: ") + cudaGetErrorString(e));
            return GDT_ERR_CUDA;
        }
    } else if (uni) {
        double *rl_coef = ws + L.rl_off, *cl_coef = rl_coef + L.runs;
        int32_t *rl_cells = reinterpret_cast<int32_t *>(cl_coef + L.runs), *cl_cells = rl_cells + L.runs;
        int32_t *rl_dst = cl_cells + L.runs, *cl_dst = rl_dst + L.runs;
        const RunListArgs rla{row_ptr, rpc, row_arc_mass, rl_cells, rl_coef, rl_dst};
        const RunListArgs cla{col_ptr, cpc, col_arc_mass, cl_cells, cl_coef, cl_dst};
        run_list_par_kernel<<<dim3(grid_size(batch * 2 * c.cells, 128), 2), 128, 0, st>>>(
            arc_off, rla, cla, kernel_w, batch, f32, c32, kappa);
        // one cluster per pair when that puts more SMs to work (see
        // ipf_cluster_kernel); GRIDOT_IPF_CLUSTER=<n> forces the cluster size
        // (1 = the single-CTA kernel), for tests and measurements
        int csz = 1;
        if (prod_smem > 0 && c.cells >= CL_MIN_UNITS && (kappa == 2 || kappa == 4 || kappa == 8)) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            csz = (int)std::max<int64_t>(1, std::min<int64_t>(CL_MAX, sms / batch));
            if (const char *e = std::getenv("GRIDOT_IPF_CLUSTER")) {
                const int v = std::atoi(e);
                if (v >= 1 && v <= CL_MAX) csz = v;
            }
        }
        bool launched = false;
        while (csz > 1 && !launched) {
            // products of one CTA's units in one batch when they fit 160 KB
            const int64_t prods = 2 * c.cells * (f.cells / c.cells);
            // (shared memory also holds 3.5 U + 2 doubles of pointers, sums and origins)
            const int64_t room = (184 * 1024) / 8 - (3 * c.cells + 2 + (c.cells + 1) / 2);
            const int cap = (int)(std::min<int64_t>(
                                      room, std::min<int64_t>(20480, ((prods / csz + 4095) / 2048) * 2048 +
                                                                         CL_SKEW * c.cells)) &
                                  ~1ll);
            if (cap < 2048) break;  // coarse grid too large for this layout: single-CTA kernel
            // products | CSR + CSC pointers | unit sums, reciprocals (f64) | block origins (i32)
            const size_t cdyn = sizeof(double) * (size_t)(cap + (c.cells + 2) + 2 * c.cells) +
                                sizeof(int32_t) * (size_t)c.cells;
            cudaFuncSetAttribute(ipf_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)cdyn);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(batch * csz));
            cfg.blockDim = dim3(PT);
            cfg.dynamicSmemBytes = cdyn;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)csz;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            const int K1 = (int)(f.cells / c.cells / kappa);
            const cudaError_t e = cudaLaunchKernelEx(
                &cfg, ipf_cluster_kernel, mu, nu, arc_off, row_ptr, col_ptr, xi, max_iter, f32,
                c32, kappa, K1, out, status, ws, L.stride_pair, (const int32_t *)rl_cells,
                (const double *)rl_coef, (const int32_t *)cl_cells, (const double *)cl_coef,
                (const int32_t *)rl_dst, (const int32_t *)cl_dst, cap);
            if (e == cudaSuccess) launched = true;
            else {
                cudaGetLastError();  // this cluster size is not schedulable here: try a smaller one
                --csz;
            }
        }
        if (launched) {
            // (pricing and TV below read the same per-pair layout)
        } else {
        if (dyn > 48 * 1024)
            cudaFuncSetAttribute(ipf_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn);
        // chains gathering from global memory: as much L1 as the SM offers
        cudaFuncSetAttribute(ipf_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             use_smem ? -1 : 0);
        ipf_kernel<true><<<(unsigned)batch, PT, dyn, st>>>(
            mu, nu, arc_off, row_ptr, row_arc_col, row_arc_mass, col_ptr, col_arc_row,
            col_arc_mass, kernel_w, xi, max_iter, f32, c32, kappa, out, status, ws, L.stride_pair,
            rpc, cpc, use_smem, bmap, rl_cells, rl_coef, cl_cells, cl_coef, prod_smem);
        }
    } else {
        if (dyn > 48 * 1024)
            cudaFuncSetAttribute(ipf_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn);
        ipf_kernel<false><<<(unsigned)batch, PT, dyn, st>>>(
            mu, nu, arc_off, row_ptr, row_arc_col, row_arc_mass, col_ptr, col_arc_row,
            col_arc_mass, kernel_w, xi, max_iter, f32, c32, kappa, out, status, ws, L.stride_pair,
            rpc, cpc, use_smem, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    }
    const int closed = uni && p == 2.0;
    int32_t *arc_row = reinterpret_cast<int32_t *>(ws + L.ar_off);
    if (!closed)
        arc_rows_kernel<<<grid_size(batch * c.cells, 256), 256, 0, st>>>(arc_off, row_ptr, batch,
                                                                         (int)c.cells, arc_row);
    dim3 gtv((unsigned)L.tv_ctas, (unsigned)batch), gpr((unsigned)L.pr_ctas, (unsigned)batch);
    if (uni) {
        auto mtv = [&](auto kern) {
            kern<<<gtv, MT, 0, st>>>(mu, nu, out, status, ws, L.stride_pair, ws + L.mom_off,
                                     ws + L.tv_off, f32, c32, kappa, p, closed, tv_lanes(f, c),
                                     tv_w);
        };
        if (ndim == 2 && kappa == 4) mtv(moments_tv_kernel<true, 2, 4>);
        else if (ndim == 2 && kappa == 8) mtv(moments_tv_kernel<true, 2, 8>);
        else if (ndim == 3 && kappa == 4) mtv(moments_tv_kernel<true, 3, 4>);
        else if (ndim == 2 && kappa == 2) mtv(moments_tv_kernel<true, 2, 2>);
        else if (ndim == 3 && kappa == 2) mtv(moments_tv_kernel<true, 3, 2>);
        else mtv(moments_tv_kernel<true, 0, 0>);
        price_kernel<true><<<gpr, MT, 0, st>>>(arc_off, row_ptr, row_arc_col, row_arc_mass,
                                               kernel_w, out, status, ws, L.stride_pair,
                                               ws + L.mom_off, ws + L.pr_off, f32, c32, kappa, p,
                                               cost_table, closed, mode == GDT_MODE_FAST,
                                               closed ? nullptr : arc_row);
    } else {
        moments_tv_kernel<false, 0, 0><<<gtv, MT, 0, st>>>(mu, nu, out, status, ws,
                                                           L.stride_pair, ws + L.mom_off,
                                                           ws + L.tv_off, f32, c32, kappa, p, 0,
                                                           tv_lanes(f, c), tv_w);
        price_kernel<false><<<gpr, MT, 0, st>>>(arc_off, row_ptr, row_arc_col, row_arc_mass,
                                                kernel_w, out, status, ws, L.stride_pair,
                                                ws + L.mom_off, ws + L.pr_off, f32, c32, kappa, p,
                                                cost_table, 0, mode == GDT_MODE_FAST, arc_row);
    }
    finish_kernel<<<grid_size(batch * 32, 128), 128, 0, st>>>(ws + L.tv_off, (int)L.tv_ctas,
                                                         ws + L.pr_off, (int)L.pr_ctas, status,
                                                         out, batch);
    return cuda_status("gdt_primal_upscale");
}

extern "C" int gdt_ipf_csr(const int64_t *indptr, const int32_t *indices, const double *data,
                           const int64_t *t_indptr, const int32_t *t_indices, const double *t_data,
                           const double *mu, const double *nu, int64_t nr, int64_t nc, double xi,
                           int64_t max_iter, double *out_a, double *out_b, double *out_kb,
                           double *out_kta, double *info, int32_t *status, void *stream) {
    GDT_CHECK_ARG(nr >= 1 && nc >= 1 && max_iter >= 1, "gdt_ipf_csr: bad sizes");
    csr_ipf_kernel<<<1, PT, 0, as_stream(stream)>>>(indptr, indices, data, t_indptr, t_indices,
                                                    t_data, mu, nu, nr, nc, xi, max_iter, out_a,
                                                    out_b, out_kb, out_kta, info, status);
    return cuda_status("gdt_ipf_csr");
}

extern "C" int gdt_price_coo(const int64_t *row, const int64_t *col, const double *mass,
                             int64_t nnz, const double *a, const double *b,
                             const double *cost_table, int64_t max_sq, double p, int ndim,
                             const int64_t *dims, double *out, void *stream) {
    Grid f;
    GDT_CHECK_ARG(make_grid(f, ndim, dims) && p >= 1.0, "gdt_price_coo: bad grid");
    (void)max_sq;
    cudaStream_t st = as_stream(stream);
    if (nnz == 0) {
        cudaMemsetAsync(out, 0, sizeof(double), st);
        return cuda_status("gdt_price_coo");
    }
    unsigned g = grid_size(nnz, 256);
    if (g > 1184) g = 1184;
    double *part = nullptr;
    if (malloc_async(reinterpret_cast<void **>(&part), sizeof(double) * g, st) != cudaSuccess)
        return cuda_status("gdt_price_coo: workspace");
    price_coo_kernel<<<g, 256, 0, st>>>(row, col, mass, nnz, a, b, cost_table, p, f, part);
    sum_parts_kernel<<<1, 32, 0, st>>>(part, (int)g, out);
    cudaFreeAsync(part, st);
    return cuda_status("gdt_price_coo");
}


#ifdef GDT_IPF_TRACE
extern "C" int gdt_debug_ex_trace(long long *host) {
    return cudaMemcpyFromSymbol(host, gdt::g_ex_trace, sizeof(long long) * 16) == cudaSuccess
               ? 0
               : -1;
}

extern "C" int gdt_debug_ipf_trace(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, gdt::g_ipf_trace, sizeof(unsigned long long) * 128) ==
                   cudaSuccess
               ? 0
               : -1;
}
#endif
