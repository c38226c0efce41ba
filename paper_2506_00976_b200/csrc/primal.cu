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
// columns of the CSR row are the cells of the arcs' target blocks in
// ascending fine flat index; `walk` enumerates exactly that order from the
// sorted arc list (lexicographic over (l_{d-1}, s_{d-1}, ..., l_0, s_0)).
// With the uniform kernel every row of block k has the same term sequence,
// so one sequential fp64 sum per coarse block replaces kappa^d row sums and
// the result is bit-identical to scipy's.  Non-uniform kernels get one sum per
// fine row (W[t,s] differs by row offset t).
//
// One CTA per pair stays resident for all sweeps (persistent over sweeps); a
// sweep is two barrier-separated phases:
//   C: per column unit l: kta = sum coef * a_i (ascending rows), then for
//      its cells b_j = nu_j / kta, gap_nu, range(b), zero-column check;
//   R: per row unit k:    kb  = sum coef * b_j (ascending columns), then for
//      its cells gap_mu with the current a, range(a), next a = mu / kb,
//      zero-row check for the next sweep.
// followed by one block reduction that applies the reference's checks in its
// order (sinkhorn.py:125-141).
#include "common.cuh"

namespace gdt {

constexpr int PT = 512;  // threads per pair CTA

__device__ __forceinline__ int64_t coord_of(int64_t id, const Grid &c, int a) {
    return (id / c.stride[a]) % c.n[a];
}

// Visit the cells of the union of coarse blocks ids[lo..hi) (sorted
// ascending) in ascending fine flat order: fn(q, cell, s) with q the arc index,
// cell the fine flat id and s the within-block offset (Fortran-flattened).
template <int LEVEL, class F>
__device__ __forceinline__ void walk(const int32_t *ids, int lo, int hi, const Grid &c,
                                     const Grid &f, int kappa, int64_t fbase, int sbase,
                                     int kpow, F &fn) {
    if constexpr (LEVEL == 0) {
        for (int q = lo; q < hi; ++q) {
            const int64_t cell = fbase + (int64_t)(ids[q] % c.n[0]) * kappa;
            for (int s0 = 0; s0 < kappa; ++s0) fn(q, cell + s0, sbase + s0);
        }
    } else {
        int r = lo;
        while (r < hi) {
            const int64_t cr = coord_of(ids[r], c, LEVEL);
            int e = r + 1;
            while (e < hi && coord_of(ids[e], c, LEVEL) == cr) ++e;
            for (int sa = 0; sa < kappa; ++sa)
                walk<LEVEL - 1>(ids, r, e, c, f, kappa, fbase + (cr * kappa + sa) * f.stride[LEVEL],
                                sbase + sa * kpow, kpow / kappa, fn);
            r = e;
        }
    }
}

template <class F>
__device__ __forceinline__ void walk_blocks(const int32_t *ids, int cnt, const Grid &c,
                                            const Grid &f, int kappa, F &fn) {
    const int top = c.nd - 1;
    const int kpow = (int)ipow(kappa, top);
    switch (c.nd) {
        case 1: walk<0>(ids, 0, cnt, c, f, kappa, 0, 0, kpow, fn); break;
        case 2: walk<1>(ids, 0, cnt, c, f, kappa, 0, 0, kpow, fn); break;
        case 3: walk<2>(ids, 0, cnt, c, f, kappa, 0, 0, kpow, fn); break;
        default: walk<3>(ids, 0, cnt, c, f, kappa, 0, 0, kpow, fn); break;
    }
}

// fine flat id of (block k, offset t)
__device__ __forceinline__ int64_t cell_of(int64_t k, int t, const Grid &c, const Grid &f,
                                           int kappa) {
    int64_t off = 0;
    for (int a = 0; a < c.nd; ++a) {
        const int64_t ka = coord_of(k, c, a);
        const int ta = t % kappa;
        t /= kappa;
        off += (ka * kappa + ta) * f.stride[a];
    }
    return off;
}

struct PairPtrs {
    const double *mu, *nu;
    const int32_t *rptr, *rcol, *cptr, *crow;
    const double *rmass, *cmass;
    double *aA, *aB, *b, *kb, *kta;
};

struct Red {  // per-sweep reduction slots
    double gap, amin, amax, bmin, bmax;
    int zrow, zcol, nonfinite;
};

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
    // sum gap, min amin/bmin, max amax/bmax, or flags; all threads get result
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r.gap += __shfl_xor_sync(0xffffffffu, r.gap, o);
        r.amin = fmin(r.amin, __shfl_xor_sync(0xffffffffu, r.amin, o));
        r.bmin = fmin(r.bmin, __shfl_xor_sync(0xffffffffu, r.bmin, o));
        r.amax = fmax(r.amax, __shfl_xor_sync(0xffffffffu, r.amax, o));
        r.bmax = fmax(r.bmax, __shfl_xor_sync(0xffffffffu, r.bmax, o));
        r.zrow |= __shfl_xor_sync(0xffffffffu, r.zrow, o);
        r.zcol |= __shfl_xor_sync(0xffffffffu, r.zcol, o);
        r.nonfinite |= __shfl_xor_sync(0xffffffffu, r.nonfinite, o);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int NW = PT / 32;
    __syncthreads();
    if (lane == 0) {
        sh[w * 8 + 0] = r.gap;
        sh[w * 8 + 1] = r.amin;
        sh[w * 8 + 2] = r.amax;
        sh[w * 8 + 3] = r.bmin;
        sh[w * 8 + 4] = r.bmax;
        sh[w * 8 + 5] = (double)(r.zrow | (r.zcol << 1) | (r.nonfinite << 2));
    }
    __syncthreads();
    Red o{0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0, 0, 0};
    for (int i = 0; i < NW; ++i) {
        o.gap += sh[i * 8 + 0];
        o.amin = fmin(o.amin, sh[i * 8 + 1]);
        o.amax = fmax(o.amax, sh[i * 8 + 2]);
        o.bmin = fmin(o.bmin, sh[i * 8 + 3]);
        o.bmax = fmax(o.bmax, sh[i * 8 + 4]);
        const int fl = (int)sh[i * 8 + 5];
        o.zrow |= fl & 1;
        o.zcol |= (fl >> 1) & 1;
        o.nonfinite |= (fl >> 2) & 1;
    }
    r = o;
    __syncthreads();
}

// Phase R for one row unit.  UNIFORM: unit = coarse block k (all its rows
// share the sum); otherwise unit = fine row (k, t).
template <bool UNIFORM>
__device__ __forceinline__ void row_unit(int64_t u, const PairPtrs &P, const Grid &c,
                                         const Grid &f, int kappa, int m, const double *W,
                                         double Wu, bool init, const double *a_cur,
                                         double *a_next, Red &r) {
    const int64_t k = UNIFORM ? u : u / m;
    const int t = UNIFORM ? 0 : (int)(u % m);
    const int lo = P.rptr[k], hi = P.rptr[k + 1];
    const int32_t *ids = P.rcol + lo;
    const double *ms = P.rmass + lo;
    double acc = 0.0;
    auto fn = [&](int q, int64_t cell, int s) {
        const double coef = __dmul_rn(ms[q], UNIFORM ? Wu : W[t * m + s]);
        acc = __dadd_rn(acc, __dmul_rn(coef, P.b[cell]));
    };
    walk_blocks(ids, hi - lo, c, f, kappa, fn);
    P.kb[u] = acc;
    const int t_lo = UNIFORM ? 0 : t, t_hi = UNIFORM ? m : t + 1;
    for (int tt = t_lo; tt < t_hi; ++tt) {
        const int64_t i = cell_of(k, tt, c, f, kappa);
        const double mui = P.mu[i];
        if (!init) {
            const double ai = a_cur[i];
            range_acc(ai, r.amin, r.amax, r.nonfinite);
            // reference gap uses support rows only; off-support a = 0, mu = 0
            if (mui > 0.0) r.gap += fabs(__dsub_rn(__dmul_rn(ai, acc), mui));
        }
        double an = 0.0;
        if (mui > 0.0) {
            if (acc <= 0.0) r.zrow = 1;
            else an = __ddiv_rn(mui, acc);
        }
        a_next[i] = an;
    }
}

template <bool UNIFORM>
__device__ __forceinline__ void col_unit(int64_t u, const PairPtrs &P, const Grid &c,
                                         const Grid &f, int kappa, int m, const double *W,
                                         double Wu, const double *a_cur, Red &r) {
    const int64_t l = UNIFORM ? u : u / m;
    const int s = UNIFORM ? 0 : (int)(u % m);
    const int lo = P.cptr[l], hi = P.cptr[l + 1];
    const int32_t *ids = P.crow + lo;
    const double *ms = P.cmass + lo;
    double acc = 0.0;
    auto fn = [&](int q, int64_t cell, int t) {
        const double coef = __dmul_rn(ms[q], UNIFORM ? Wu : W[t * m + s]);
        acc = __dadd_rn(acc, __dmul_rn(coef, a_cur[cell]));
    };
    walk_blocks(ids, hi - lo, c, f, kappa, fn);
    P.kta[u] = acc;
    const int s_lo = UNIFORM ? 0 : s, s_hi = UNIFORM ? m : s + 1;
    for (int ss = s_lo; ss < s_hi; ++ss) {
        const int64_t j = cell_of(l, ss, c, f, kappa);
        const double nuj = P.nu[j];
        double bj = 0.0;
        if (nuj > 0.0) {
            if (acc <= 0.0) r.zcol = 1;
            else bj = __ddiv_rn(nuj, acc);
            range_acc(bj, r.bmin, r.bmax, r.nonfinite);
            r.gap += fabs(__dsub_rn(nuj, __dmul_rn(bj, acc)));
        }
        P.b[j] = bj;
    }
}

__device__ __forceinline__ double grid_cost(int64_t i, int64_t j, const Grid &f, double p,
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

__device__ __forceinline__ double tv_weight(int64_t i, const Grid &f, double p) {
    double parts[GDT_MAX_DIM];
    for (int a = f.nd - 1; a >= 0; --a) {
        const int64_t x = i / f.stride[a];
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

template <bool UNIFORM>
__global__ void __launch_bounds__(PT) primal_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const int64_t *__restrict__ arc_off,
    const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ row_arc_col,
    const double *__restrict__ row_arc_mass, const int32_t *__restrict__ col_ptr,
    const int32_t *__restrict__ col_arc_row, const double *__restrict__ col_arc_mass,
    const double *__restrict__ W, const double *__restrict__ xi_in, int64_t max_iter, double p,
    Grid f, Grid c, int kappa, const double *__restrict__ table, double *__restrict__ out,
    int32_t *__restrict__ status, double *__restrict__ scratch) {
    __shared__ double sh[(PT / 32) * 8];
    const int64_t b = blockIdx.x;
    const int64_t N = f.cells, n = c.cells;
    const int m = (int)ipow(kappa, f.nd);
    const int64_t U = UNIFORM ? n : N;
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
    double *ws = scratch + b * (3 * N + 2 * U);
    P.aA = ws;
    P.aB = ws + N;
    P.b = ws + 2 * N;
    P.kb = ws + 3 * N;
    P.kta = ws + 3 * N + U;

    // supports and the reference's default xi (quantized.py:317-320)
    double cnt = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += PT) {
        const double mi = P.mu[i], ni = P.nu[i];
        cnt += (mi > 0.0 ? 1.0 : 0.0) + (ni > 0.0 ? 1.0 : 0.0);
        P.b[i] = ni > 0.0 ? 1.0 : 0.0;  // b = ones over the target support
    }
    cnt = block_sum<PT>(cnt, sh);
    const double xi = xi_in[b] < 0.0 ? 1e-9 * cnt : xi_in[b];
    __syncthreads();

    // kb = K b0, a = mu / kb (sinkhorn.py:119-129 before the first sweep)
    Red r{0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0, 0, 0};
    double *a_cur = P.aA, *a_nxt = P.aB;
    for (int64_t u = threadIdx.x; u < U; u += PT)
        row_unit<UNIFORM>(u, P, c, f, kappa, m, W, Wu, true, nullptr, a_cur, r);
    block_reduce_red(r, sh);
    int st = r.zrow ? GDT_PAIR_ZERO_DENOM_ROW : GDT_PAIR_OK;
    int64_t it = 0;
    double gap = INFINITY;
    bool converged = false;
    while (st == GDT_PAIR_OK && it < max_iter) {
        ++it;
        Red rc{0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0, 0, 0};
        for (int64_t u = threadIdx.x; u < U; u += PT)
            col_unit<UNIFORM>(u, P, c, f, kappa, m, W, Wu, a_cur, rc);
        __syncthreads();
        // zero-column check must precede anything that reads b
        int zc = __syncthreads_or(rc.zcol);
        if (zc) {
            st = GDT_PAIR_ZERO_DENOM_COL;
            break;
        }
        for (int64_t u = threadIdx.x; u < U; u += PT)
            row_unit<UNIFORM>(u, P, c, f, kappa, m, W, Wu, false, a_cur, a_nxt, rc);
        block_reduce_red(rc, sh);
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
        if (rc.zrow) {  // checked at the top of the next sweep
            st = GDT_PAIR_ZERO_DENOM_ROW;
            break;
        }
        double *tmp = a_cur;
        a_cur = a_nxt;
        a_nxt = tmp;
    }
    // on exit a_cur / b / kb / kta are the state of the last completed sweep
    if (threadIdx.x == 0) status[b] = st;
    if (st != GDT_PAIR_OK) {
        if (threadIdx.x == 0) {
            for (int q = 0; q < 8; ++q) out[b * 8 + q] = 0.0;
            out[b * 8 + 4] = (double)it;
        }
        return;
    }

    // pricing: sum over fine entries of ((a_i * m W_ts) * b_j) * C_ij
    // (quantized.py:346-355; order-free like the reference's BLAS dot)
    double price = 0.0;
    const int64_t A = P.rptr[n];
    for (int64_t w = threadIdx.x; w < A * m; w += PT) {
        const int64_t q = w / m;
        const int t = (int)(w - q * m);
        // arc q in row-major order: find its row block by binary search
        int lo = 0, hi = (int)n;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (P.rptr[mid] <= q) lo = mid;
            else hi = mid;
        }
        const int64_t k = lo, l = P.rcol[q];
        const double mass = P.rmass[q];
        const int64_t i = cell_of(k, t, c, f, kappa);
        const double ai = a_cur[i];
        if (ai == 0.0) continue;
        for (int s = 0; s < m; ++s) {
            const int64_t j = cell_of(l, s, c, f, kappa);
            const double wts = UNIFORM ? Wu : W[t * m + s];
            const double fitted = __dmul_rn(__dmul_rn(ai, __dmul_rn(mass, wts)), P.b[j]);
            price += fitted * grid_cost(i, j, f, p, table);
        }
    }
    price = block_sum<PT>(price, sh);

    // weighted TV inner sums with mu_hat = a * kb, nu_hat = b * kta
    double tmu = 0.0, tnu = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += PT) {
        const double w = tv_weight(i, f, p);
        // unit of cell i: its block k (uniform) or the fine row/column (k, t)
        int64_t rem = i, k = 0, t = 0, tpow = 1;
        for (int a = f.nd - 1; a >= 0; --a) {
            const int64_t x = rem / f.stride[a];
            rem -= x * f.stride[a];
            k += (x / kappa) * c.stride[a];
        }
        for (int a = 0; a < f.nd; ++a) {
            const int64_t x = (i / f.stride[a]) % f.n[a];
            t += (x % kappa) * tpow;
            tpow *= kappa;
        }
        const int64_t unit = UNIFORM ? k : k * m + t;
        const double mh = P.mu[i] > 0.0 ? __dmul_rn(a_cur[i], P.kb[unit]) : 0.0;
        const double nh = P.nu[i] > 0.0 ? __dmul_rn(P.b[i], P.kta[unit]) : 0.0;
        tmu += w * fabs(__dsub_rn(mh, P.mu[i]));
        tnu += w * fabs(__dsub_rn(nh, P.nu[i]));
    }
    tmu = block_sum<PT>(tmu, sh);
    tnu = block_sum<PT>(tnu, sh);
    if (threadIdx.x == 0) {
        double *o = out + b * 8;
        o[0] = price;
        o[1] = tmu;
        o[2] = tnu;
        o[3] = gap;
        o[4] = (double)it;
        o[5] = converged ? 1.0 : 0.0;
        o[6] = cnt;
        o[7] = 0.0;
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
    double *__restrict__ kb, double *__restrict__ kta, double *__restrict__ a_prev,
    double *__restrict__ info, int32_t *__restrict__ status) {
    __shared__ double sh[(PT / 32) * 8];
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
        Red r{0.0, INFINITY, -INFINITY, INFINITY, -INFINITY, 0, 0, 0};
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
        const bool bad_a = r.amin <= r.amax && (r.amin < 1e-100 || r.amax > 1e100 || !isfinite(r.amax));
        const bool bad_b = r.bmin <= r.bmax && (r.bmin < 1e-100 || r.bmax > 1e100 || !isfinite(r.bmax));
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
    (void)a_prev;
    if (threadIdx.x == 0) {
        info[0] = (double)it;
        info[1] = gap;
        info[2] = conv ? 1.0 : 0.0;
        info[3] = 0.0;
        status[0] = st;
    }
}

__global__ void price_coo_kernel(const int64_t *__restrict__ row, const int64_t *__restrict__ col,
                                 const double *__restrict__ mass, int64_t nnz,
                                 const double *__restrict__ a, const double *__restrict__ b,
                                 const double *__restrict__ table, double p, Grid f,
                                 double *__restrict__ out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double fitted = __dmul_rn(__dmul_rn(a[row[e]], mass[e]), b[col[e]]);
        acc += fitted * grid_cost(row[e], col[e], f, p, table);
    }
    acc = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) atomicAdd(out, acc);
}

}  // namespace gdt

using namespace gdt;

extern "C" int64_t gdt_primal_scratch_bytes(int64_t batch, int ndim, const int64_t *dims,
                                            int kappa, int kernel_uniform) {
    Grid f, c;
    if (!make_grid(f, ndim, dims) || !make_coarse(c, f, kappa)) return -1;
    const int64_t U = kernel_uniform ? c.cells : f.cells;
    return (int64_t)sizeof(double) * batch * (3 * f.cells + 2 * U);
}

extern "C" int gdt_primal_upscale(const double *mu, const double *nu, const int64_t *arc_off,
                                        const int32_t *row_ptr, const int32_t *row_arc_col,
                                        const double *row_arc_mass, const int32_t *col_ptr,
                                        const int32_t *col_arc_row, const double *col_arc_mass,
                                        const double *kernel_w, int kernel_uniform,
                                        const double *xi, int64_t max_iter, double p,
                                        int64_t batch, int ndim, const int64_t *dims, int kappa,
                                        const double *cost_table, int64_t max_sq, double *out,
                                        int32_t *status, void *scratch, void *stream) {
    Grid f, c;
    GDT_CHECK_ARG(make_grid(f, ndim, dims) && make_coarse(c, f, kappa),
                  "gdt_primal_upscale: dims must be positive multiples of kappa");
    GDT_CHECK_ARG(p >= 1.0 && max_iter >= 1 && batch >= 0, "gdt_primal_upscale: bad p/max_iter");
    int64_t need_sq = 0;
    for (int a = 0; a < ndim; ++a) need_sq += (dims[a] - 1) * (dims[a] - 1);
    GDT_CHECK_ARG(p == 1.0 || p == 2.0 || (cost_table != nullptr && max_sq >= need_sq),
                  "gdt_primal_upscale: cost_table required for p not in {1, 2}");
    if (batch == 0) return GDT_OK;
    cudaStream_t st = as_stream(stream);
    if (kernel_uniform)
        primal_kernel<true><<<(unsigned)batch, PT, 0, st>>>(
            mu, nu, arc_off, row_ptr, row_arc_col, row_arc_mass, col_ptr, col_arc_row, col_arc_mass,
            kernel_w, xi, max_iter, p, f, c, kappa, cost_table, out, status, (double *)scratch);
    else
        primal_kernel<false><<<(unsigned)batch, PT, 0, st>>>(
            mu, nu, arc_off, row_ptr, row_arc_col, row_arc_mass, col_ptr, col_arc_row, col_arc_mass,
            kernel_w, xi, max_iter, p, f, c, kappa, cost_table, out, status, (double *)scratch);
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
                                                    out_b, out_kb, out_kta, nullptr, info, status);
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
    cudaMemsetAsync(out, 0, sizeof(double), st);
    if (nnz == 0) return cuda_status("gdt_price_coo");
    unsigned g = grid_size(nnz, 256);
    if (g > 1184) g = 1184;
    price_coo_kernel<<<g, 256, 0, st>>>(row, col, mass, nnz, a, b, cost_table, p, f, out);
    return cuda_status("gdt_price_coo");
}
