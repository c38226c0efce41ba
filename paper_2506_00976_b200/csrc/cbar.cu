// K2: marginally weighted coarse cost C-bar (costs.py:128-171).
//
// Exact mode restates the reference's numpy order bit for bit:
//   s_{k,c} = sequential over the block's rows r (ascending fine index) of
//             (C_rc * mu_r) * nu_c                       (costs.py:158-162)
//   numer_kl = numpy pairwise sum of s_{k,c} over c in Y_l (ascending)
//   C-bar_kl = numer_kl / (mu~_k * nu~_l), or C-tilde_kl where that is 0.
// A CTA owns (pair, KT row blocks, LT column blocks); each thread owns
// column cells, keeps the KT partial sums in registers/shared memory, and the
// pairwise block sums are formed from shared memory.  Products use
// __dmul_rn/__dadd_rn so no FMA contraction can change the rounding.
//
// Fast mode (the fp32 mode of BASELINE.json): p == 2 uses block moments --
// sum_{r,c} |x_r - y_c|^2 mu_r nu_c expands into per-block 0th/1st/2nd
// moments about the block centres, O(N^d + n^2d) instead of O(N^2d) -- and
// other p use the same tiling as exact mode in fp32 FFMA with an fp64 block
// sum.
#include <algorithm>

#include "common.cuh"

namespace gdt {

int cbar_fast_diag(const double *mu, const double *nu, const double *mu_c, const double *nu_c,
                   const double *Ccentre, const double *table, int64_t max_sq, double *out,
                   uint8_t *unused, int64_t batch, const Grid &f, const Grid &c, int kappa, double p,
                   cudaStream_t st);
int cbar_fast_toeplitz(const double *mu, const double *nu, const double *mu_c,
                       const double *nu_c, const double *Ccentre, const double *table,
                       int64_t max_sq, double *out, uint8_t *unused, int64_t batch, const Grid &f,
                       const Grid &c, int kappa, double p, cudaStream_t st);

struct Offsets {  // within-block offset vectors t -> (t_0..t_{d-1})
    int8_t v[GDT_MAX_DIM];
};

__device__ __forceinline__ void unravel_block(int64_t id, const Grid &c, int64_t *out) {
    for (int a = c.nd - 1; a >= 0; --a) {
        out[a] = id / c.stride[a];
        id -= out[a] * c.stride[a];
    }
}

template <bool EXACT>
__global__ void __launch_bounds__(256) cbar_tile_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const double *__restrict__ mu_c,
    const double *__restrict__ nu_c, const double *__restrict__ Ccentre,
    const double *__restrict__ table, double *__restrict__ out, uint8_t *__restrict__ unused,
    Grid f, Grid c, int kappa, int m, double p, int KT, int LT) {
    extern __shared__ double smem[];
    using T = typename std::conditional<EXACT, double, float>::type;
    const int cols = LT * m;
    T *S = reinterpret_cast<T *>(smem);                       // [KT][cols]
    double *mus = smem + (KT * cols * sizeof(T) + 7) / 8;     // [KT][m]
    int *roff = reinterpret_cast<int *>(mus + KT * m);        // [m][nd] offsets

    const int64_t b = blockIdx.z;
    const int64_t k0 = (int64_t)blockIdx.y * KT, l0 = (int64_t)blockIdx.x * LT;
    const int64_t n = c.cells;
    const double *mub = mu + b * f.cells, *nub = nu + b * f.cells;

    for (int t = threadIdx.x; t < m; t += blockDim.x) {
        int rem = t;
        for (int a = 0; a < f.nd; ++a) {
            roff[t * GDT_MAX_DIM + a] = rem % kappa;
            rem /= kappa;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < KT * m; i += blockDim.x) {
        const int kk = i / m, t = i - kk * m;
        const int64_t k = k0 + kk;
        double v = 0.0;
        if (k < n) {
            int64_t kc[GDT_MAX_DIM];
            unravel_block(k, c, kc);
            int64_t off = 0;
            for (int a = 0; a < f.nd; ++a) off += (kc[a] * kappa + roff[t * GDT_MAX_DIM + a]) * f.stride[a];
            v = mub[off];
        }
        mus[i] = v;
    }
    __syncthreads();

    for (int cl = threadIdx.x; cl < cols; cl += blockDim.x) {
        const int64_t l = l0 + cl / m;
        const int s = cl % m;
        if (l >= n) {
            for (int kk = 0; kk < KT; ++kk) S[kk * cols + cl] = (T)0;
            continue;
        }
        int64_t lc[GDT_MAX_DIM], xc[GDT_MAX_DIM];
        unravel_block(l, c, lc);
        int64_t coff = 0;
        for (int a = 0; a < f.nd; ++a) {
            xc[a] = lc[a] * kappa + roff[s * GDT_MAX_DIM + a];
            coff += xc[a] * f.stride[a];
        }
        const double nuc = nub[coff];
        for (int kk = 0; kk < KT; ++kk) {
            const int64_t k = k0 + kk;
            if (k >= n) {
                S[kk * cols + cl] = (T)0;
                continue;
            }
            int64_t kc[GDT_MAX_DIM];
            unravel_block(k, c, kc);
            int64_t base[GDT_MAX_DIM];
            for (int a = 0; a < f.nd; ++a) base[a] = kc[a] * kappa - xc[a];
            if (EXACT) {
                double acc = 0.0;
                for (int t = 0; t < m; ++t) {
                    int64_t sq = 0;
                    for (int a = 0; a < f.nd; ++a) {
                        const int64_t dd = base[a] + roff[t * GDT_MAX_DIM + a];
                        sq += dd * dd;
                    }
                    const double cost = cost_from_sq(sq, p, table);
                    const double term = __dmul_rn(__dmul_rn(cost, mus[kk * m + t]), nuc);
                    acc = t == 0 ? term : __dadd_rn(acc, term);
                }
                S[kk * cols + cl] = (T)acc;
            } else {
                float acc = 0.0f;
                for (int t = 0; t < m; ++t) {
                    int sq = 0;
                    for (int a = 0; a < f.nd; ++a) {
                        const int dd = (int)base[a] + roff[t * GDT_MAX_DIM + a];
                        sq += dd * dd;
                    }
                    const float cost = p == 2.0 ? (float)sq
                                       : p == 1.0 ? __fsqrt_rn((float)sq)
                                                  : (float)table[sq];
                    acc = fmaf(cost, (float)mus[kk * m + t], acc);
                }
                S[kk * cols + cl] = (T)(acc * (float)nuc);
            }
        }
    }
    __syncthreads();

    for (int o = threadIdx.x; o < KT * LT; o += blockDim.x) {
        const int kk = o / LT, ll = o - kk * LT;
        const int64_t k = k0 + kk, l = l0 + ll;
        if (k >= n || l >= n) continue;
        const T *row = S + kk * cols + ll * m;
        double numer;
        if (EXACT) {
            numer = np_pairwise([&](int64_t i) { return (double)row[i]; }, m);
        } else {
            numer = 0.0;
            for (int i = 0; i < m; ++i) numer += (double)row[i];
        }
        const double denom = __dmul_rn(mu_c[b * n + k], nu_c[b * n + l]);
        const int64_t oi = (b * n + k) * n + l;
        const bool un = denom == 0.0;
        out[oi] = un ? Ccentre[k * n + l] : __ddiv_rn(numer, denom);
        if (unused) unused[oi] = un ? 1 : 0;
    }
}

// ---- exact mode, p != 2, 2-D / 3-D grids: one row block per CTA ----------
// The same arithmetic as cbar_tile_kernel<true> (the reference's order:
// s_kc = sequential over t of (C_tc * mu_t) * nu_c, then the numpy pairwise
// sum over c in Y_l), organised for throughput: a CTA owns ONE row block k
// (its mu_t in shared memory) and a chunk of target blocks; each thread runs
// the chain of one target cell at a time with the cost read from the
// reference-exact table by integer squared distance (incremental offsets, no
// divisions in the loop), and the chains of a chunk land in shared memory in
// fine order for the pairwise block sums.
constexpr int CE_THREADS = 256;
constexpr int CE_CELLS = 2048;  // target cells per CTA (chunk of whole blocks)

template <int KAPPA, int ND>
__global__ void __launch_bounds__(CE_THREADS) cbar_exact_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const double *__restrict__ mu_c,
    const double *__restrict__ nu_c, const double *__restrict__ Ccentre,
    const double *__restrict__ table, double p, double *__restrict__ out,
    uint8_t *__restrict__ unused, Grid f, Grid c, int LT) {
    constexpr int M = ND == 2 ? KAPPA * KAPPA : KAPPA * KAPPA * KAPPA;
    __shared__ double mus[M];
    extern __shared__ double S[];  // [LT][M] chains of the chunk, fine order per block
    const int64_t b = blockIdx.z;
    const int64_t n = c.cells;
    const int64_t k = blockIdx.x;
    const int64_t l0 = (int64_t)blockIdx.y * LT;
    const int lt = (int)(n - l0 < LT ? n - l0 : LT);
    const double *mub = mu + b * f.cells, *nub = nu + b * f.cells;
    // row block k: origin and its masses in the reference's order (t = tx + K ty (+ K^2 tz))
    int kx[3] = {0, 0, 0};
    {
        int64_t rem = k;
        for (int a = ND - 1; a >= 0; --a) {
            kx[a] = (int)(rem / c.stride[a]);
            rem -= (int64_t)kx[a] * c.stride[a];
        }
    }
    for (int t = threadIdx.x; t < M; t += CE_THREADS) {
        const int tx = t % KAPPA, ty = (t / KAPPA) % KAPPA, tz = t / (KAPPA * KAPPA);
        int64_t off = (int64_t)(kx[0] * KAPPA + tx) + (int64_t)(kx[1] * KAPPA + ty) * f.stride[1];
        if (ND == 3) off += (int64_t)(kx[2] * KAPPA + tz) * f.stride[2];
        mus[t] = mub[off];
    }
    __syncthreads();
    const int cells = lt * M;
    for (int i = threadIdx.x; i < cells; i += CE_THREADS) {
        const int ll = i / M, sidx = i - ll * M;  // target block (chunk-local), cell in it
        int64_t lrem = l0 + ll;
        int lc[3] = {0, 0, 0};
        for (int a = ND - 1; a >= 0; --a) {
            lc[a] = (int)(lrem / c.stride[a]);
            lrem -= (int64_t)lc[a] * c.stride[a];
        }
        const int sx = sidx % KAPPA, sy = (sidx / KAPPA) % KAPPA, sz = sidx / (KAPPA * KAPPA);
        const int cx = lc[0] * KAPPA + sx, cy = lc[1] * KAPPA + sy, cz = ND == 3 ? lc[2] * KAPPA + sz : 0;
        const double nuc = nub[cx + (int64_t)cy * f.stride[1] + (ND == 3 ? (int64_t)cz * f.stride[2] : 0)];
        // offsets of the row block's cells from c: dx = kx0 + tx - cx, ...
        const int dx0 = kx[0] * KAPPA - cx, dy0 = kx[1] * KAPPA - cy,
                  dz0 = ND == 3 ? kx[2] * KAPPA - cz : 0;
        double acc = 0.0;
#pragma unroll 1
        for (int tz = 0; tz < (ND == 3 ? KAPPA : 1); ++tz) {
            const int dz = dz0 + tz;
#pragma unroll 1
            for (int ty = 0; ty < KAPPA; ++ty) {
                const int dy = dy0 + ty;
                const int h = dy * dy + dz * dz;
                const double *mrow = mus + (tz * KAPPA + ty) * KAPPA;
                double cst[KAPPA];
#pragma unroll
                for (int tx = 0; tx < KAPPA; ++tx) {
                    const int dx = dx0 + tx;
                    const int sq = h + dx * dx;
                    cst[tx] = table ? __ldg(table + sq) : (p == 1.0 ? __dsqrt_rn((double)sq) : (double)sq);
                }
#pragma unroll
                for (int tx = 0; tx < KAPPA; ++tx) {
                    const double term = __dmul_rn(__dmul_rn(cst[tx], mrow[tx]), nuc);
                    acc = (tz == 0 && ty == 0 && tx == 0) ? term : __dadd_rn(acc, term);
                }
            }
        }
        S[i] = acc;
    }
    __syncthreads();
    for (int ll = threadIdx.x; ll < lt; ll += CE_THREADS) {
        const int64_t l = l0 + ll;
        const double *row = S + ll * M;
        const double numer = np_pairwise([&](int64_t i) { return row[i]; }, M);
        const double denom = __dmul_rn(mu_c[b * n + k], nu_c[b * n + l]);
        const int64_t oi = (b * n + k) * n + l;
        const bool un = denom == 0.0;
        out[oi] = un ? Ccentre[k * n + l] : __ddiv_rn(numer, denom);
        if (unused) unused[oi] = un ? 1 : 0;
    }
}

// 2-D grids: the same chains with the CTA's target cells taken in fine-row
// order (a warp = 32 consecutive cells of one fine row), so the costs a warp
// needs for one source cell are consecutive entries of a 2-D table
// T2[|dy|][|dx|] = cost(dx^2 + dy^2) -- the same doubles as the 1-D table --
// and its loads coalesce instead of scattering over the squared distances.
__global__ void cost2d_kernel(const double *__restrict__ table, double p, int W, int H,
                              double *__restrict__ t2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W * H; i += gridDim.x * blockDim.x) {
        const int a = i / W, bx = i - a * W;
        const int64_t sq = (int64_t)a * a + (int64_t)bx * bx;
        t2[i] = table ? table[sq] : (p == 1.0 ? __dsqrt_rn((double)sq) : (double)sq);
    }
}

template <int KAPPA>
__global__ void __launch_bounds__(CE_THREADS) cbar_exact2d_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const double *__restrict__ mu_c,
    const double *__restrict__ nu_c, const double *__restrict__ Ccentre,
    const double *__restrict__ t2, int W, double *__restrict__ out, uint8_t *__restrict__ unused,
    Grid f, Grid c, int BR) {
    constexpr int M = KAPPA * KAPPA;
    __shared__ double mus[M];
    extern __shared__ double S[];  // [chunk blocks][M], fine order per block
    const int64_t b = blockIdx.z;
    const int64_t n = c.cells;
    const int n0 = (int)c.n[0], N0 = (int)f.n[0];
    const int k = blockIdx.x;
    const int br0 = blockIdx.y * BR;                       // first block-row of the chunk
    const int brs = min(BR, (int)c.n[1] - br0);            // block-rows in the chunk
    const int64_t l0 = (int64_t)br0 * n0;
    const double *mub = mu + b * f.cells, *nub = nu + b * f.cells;
    const int kx = k % n0, ky = k / n0;
    for (int t = threadIdx.x; t < M; t += CE_THREADS) {
        const int tx = t % KAPPA, ty = t / KAPPA;
        mus[t] = mub[(kx * KAPPA + tx) + (int64_t)(ky * KAPPA + ty) * N0];
    }
    __syncthreads();
    const int cells = brs * KAPPA * N0;
    for (int i = threadIdx.x; i < cells; i += CE_THREADS) {
        const int cyl = i / N0, cx = i - cyl * N0;
        const int cy = br0 * KAPPA + cyl;
        const double nuc = nub[cx + (int64_t)cy * N0];
        const int dx0 = kx * KAPPA - cx, dy0 = ky * KAPPA - cy;
        double acc = 0.0;
#pragma unroll
        for (int ty = 0; ty < KAPPA; ++ty) {
            const int dy = dy0 + ty;
            const double *row = t2 + (int64_t)(dy < 0 ? -dy : dy) * W;
            double cst[KAPPA];
#pragma unroll
            for (int tx = 0; tx < KAPPA; ++tx) {
                const int dx = dx0 + tx;
                cst[tx] = __ldg(row + (dx < 0 ? -dx : dx));
            }
#pragma unroll
            for (int tx = 0; tx < KAPPA; ++tx) {
                const double term = __dmul_rn(__dmul_rn(cst[tx], mus[ty * KAPPA + tx]), nuc);
                acc = (ty == 0 && tx == 0) ? term : __dadd_rn(acc, term);
            }
        }
        // staged at (block, cell in block) for the pairwise block sums
        const int ll = (cyl / KAPPA) * n0 + cx / KAPPA;
        S[ll * M + (cx % KAPPA) + KAPPA * (cyl % KAPPA)] = acc;
    }
    __syncthreads();
    for (int ll = threadIdx.x; ll < brs * n0; ll += CE_THREADS) {
        const int64_t l = l0 + ll;
        const double *rowp = S + ll * M;
        const double numer = np_pairwise([&](int64_t i) { return rowp[i]; }, M);
        const double denom = __dmul_rn(mu_c[b * n + k], nu_c[b * n + l]);
        const int64_t oi = (b * n + k) * n + l;
        const bool un = denom == 0.0;
        out[oi] = un ? Ccentre[(int64_t)k * n + l] : __ddiv_rn(numer, denom);
        if (unused) unused[oi] = un ? 1 : 0;
    }
}

// ---- fast p == 2: block moments ------------------------------------------
// mom layout per (pair, block): [M1_0 .. M1_{d-1}, M2] about the block centre.
// ND / KAP > 0: compile-time dimension and pooling factor -- the cell loop is
// fully unrolled (all loads of a block in flight, offsets by shifts) with the
// same left-to-right summation order as the runtime version (ND = KAP = 0).
template <int ND, int KAP>
__global__ void moments_kernel(const double *__restrict__ fine, double *__restrict__ mom,
                               int64_t batch, Grid f, Grid c, int kappa_rt) {
    const int kappa = KAP ? KAP : kappa_rt;
    const int nd = ND ? ND : f.nd;
    const int64_t total = batch * c.cells;
    const int W = nd + 1;
    const double ctr = (kappa - 1) / 2.0;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / c.cells, k = idx - b * c.cells;
        int64_t kc[GDT_MAX_DIM];
        unravel_block(k, c, kc);
        int64_t origin = b * f.cells;
        for (int a = 0; a < nd; ++a) origin += kc[a] * kappa * f.stride[a];
        double m1[GDT_MAX_DIM] = {0, 0, 0, 0}, m2 = 0.0;
        if constexpr (ND > 0 && KAP > 0) {
            constexpr int M = ND == 1 ? KAP : (ND == 2 ? KAP * KAP : KAP * KAP * KAP);
            static_assert(ND <= 3, "compile-time blocks up to 3-D");
            const double *base = fine + origin;
            const int64_t s1 = f.stride[1], s2 = f.stride[2];
            double wv[M];
#pragma unroll
            for (int t = 0; t < M; ++t) {
                const int o0 = t % KAP, o1 = (t / KAP) % KAP, o2 = t / (KAP * KAP);
                wv[t] = __ldg(base + o0 + (ND > 1 ? o1 * s1 : 0) + (ND > 2 ? o2 * s2 : 0));
            }
#pragma unroll
            for (int t = 0; t < M; ++t) {
                const int o[3] = {t % KAP, (t / KAP) % KAP, t / (KAP * KAP)};
                double r2 = 0.0, dl[3];
#pragma unroll
                for (int a = 0; a < ND; ++a) {
                    dl[a] = o[a] - ctr;
                    r2 += dl[a] * dl[a];
                }
#pragma unroll
                for (int a = 0; a < ND; ++a) m1[a] += wv[t] * dl[a];
                m2 += wv[t] * r2;
            }
        } else {
            const int m = (int)ipow(kappa, nd);
            for (int t = 0; t < m; ++t) {
                int rem = t;
                int64_t off = 0;
                double r2 = 0.0, dl[GDT_MAX_DIM];
                for (int a = 0; a < nd; ++a) {
                    const int o = rem % kappa;
                    rem /= kappa;
                    off += o * f.stride[a];
                    dl[a] = o - ctr;
                    r2 += dl[a] * dl[a];
                }
                const double w = fine[origin + off];
                for (int a = 0; a < nd; ++a) m1[a] += w * dl[a];
                m2 += w * r2;
            }
        }
        double *o = mom + idx * W;
        for (int a = 0; a < nd; ++a) o[a] = m1[a];
        o[nd] = m2;
    }
}

// grid: x = chunk of 4*256 columns l, y = group of MB_K row blocks k, z =
// pair.  A thread keeps the moments of its 4 consecutive columns in registers
// and sweeps the MB_K rows, whose moments sit in shared memory; the quotient
// uses reciprocals (fp32 mode: any order / rounding within ~1e-15).  ND is a
// template parameter so the per-axis loops unroll; per output the expansion
//   numer = denom |D|^2 + 2 D.(M1_k N0_l - M0_k N1_l) + M2_k N0_l + M0_k N2_l
//           - 2 M1_k.N1_l,   D = kappa (k - l) in block units,
// is ~4 ND + 6 FP64 operations against 9 bytes written: HBM-bound.
constexpr int MB_K = 16;

template <int ND>
__global__ void __launch_bounds__(256) cbar_moments_kernel(
    const double *__restrict__ mu_c, const double *__restrict__ nu_c, const double *__restrict__ mm,
    const double *__restrict__ nm, const double *__restrict__ Ccentre, double *__restrict__ out,
    uint8_t *__restrict__ unused, Grid c, int kappa) {
    constexpr int W = ND + 1;
    __shared__ double sk[MB_K][ND + 3];  // M0, 1/M0, M1[ND], M2
    __shared__ double skd[MB_K][ND];     // kappa * k coordinates
    const int n = (int)c.cells;
    const int k0 = blockIdx.y * MB_K;
    const int64_t b = blockIdx.z;
    if (threadIdx.x < MB_K) {
        const int k = k0 + threadIdx.x;
        if (k < n) {
            const double M0 = mu_c[b * n + k];
            const double *Mk = mm + ((int64_t)b * n + k) * W;
            sk[threadIdx.x][0] = M0;
            sk[threadIdx.x][1] = M0 > 0.0 ? 1.0 / M0 : 0.0;
#pragma unroll
            for (int a = 0; a <= ND; ++a) sk[threadIdx.x][2 + a] = Mk[a];
            int kk = k;
#pragma unroll
            for (int a = 0; a < ND; ++a) {
                const int ca = kk % (int)c.n[a];
                kk /= (int)c.n[a];
                skd[threadIdx.x][a] = (double)(kappa * ca);
            }
        }
    }
    __syncthreads();
    const int l0 = (blockIdx.x * 256 + threadIdx.x) * 4;
    if (l0 >= n) return;
    double N0[4], iN[4], N1[4][ND], N2[4], ld[4][ND];
    {
        int cc[ND];
        int ll = l0;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
            cc[a] = ll % (int)c.n[a];
            ll /= (int)c.n[a];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int l = l0 + q < n ? l0 + q : n - 1;
            N0[q] = nu_c[b * n + l];
            iN[q] = N0[q] > 0.0 ? 1.0 / N0[q] : 0.0;
            const double *Nl = nm + ((int64_t)b * n + l) * W;
#pragma unroll
            for (int a = 0; a < ND; ++a) {
                N1[q][a] = Nl[a];
                ld[q][a] = (double)(kappa * cc[a]);
            }
            N2[q] = Nl[ND];
            ++cc[0];
#pragma unroll
            for (int a = 0; a < ND - 1; ++a)
                if (cc[a] >= (int)c.n[a]) {
                    cc[a] = 0;
                    ++cc[a + 1];
                }
        }
    }
    const bool vec = l0 + 3 < n && (n & 3) == 0;
    const int kend = min(MB_K, n - k0);
    for (int kk = 0; kk < kend; ++kk) {
        const int k = k0 + kk;
        const double M0 = sk[kk][0], iM = sk[kk][1], M2 = sk[kk][2 + ND];
        const int64_t orow = ((int64_t)b * n + k) * n;
        double vals[4];
        uint8_t un[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double denom = __dmul_rn(M0, N0[q]);
            double d2 = 0.0, cross = 0.0, m1n1 = 0.0;
#pragma unroll
            for (int a = 0; a < ND; ++a) {
                const double D = skd[kk][a] - ld[q][a];
                const double M1 = sk[kk][2 + a];
                d2 = fma(D, D, d2);
                cross = fma(D, M1 * N0[q] - M0 * N1[q][a], cross);
                m1n1 = fma(M1, N1[q][a], m1n1);
            }
            const double numer = denom * d2 + 2.0 * cross + M2 * N0[q] + M0 * N2[q] - 2.0 * m1n1;
            un[q] = denom == 0.0;
            vals[q] = numer * iM * iN[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (un[q]) vals[q] = l0 + q < n ? Ccentre[(int64_t)k * n + l0 + q] : 0.0;
        if (vec) {
            reinterpret_cast<double2 *>(out + orow + l0)[0] = make_double2(vals[0], vals[1]);
            reinterpret_cast<double2 *>(out + orow + l0)[1] = make_double2(vals[2], vals[3]);
            if (unused)
                *reinterpret_cast<uchar4 *>(unused + orow + l0) =
                    make_uchar4(un[0], un[1], un[2], un[3]);
        } else {
            for (int q = 0; q < 4 && l0 + q < n; ++q) {
                out[orow + l0 + q] = vals[q];
                if (unused) unused[orow + l0 + q] = un[q];
            }
        }
    }
}

}  // namespace gdt

using namespace gdt;

extern "C" int gdt_weighted_cost(const double *mu, const double *nu, const double *mu_c,
                                 const double *nu_c, const double *centre_cost,
                                 const double *cost_table, int64_t max_sq, double *out,
                                 uint8_t *unused, int64_t batch, int ndim, const int64_t *dims,
                                 int kappa, double p, int mode, void *stream) {
    Grid f, c;
    GDT_CHECK_ARG(make_grid(f, ndim, dims) && make_coarse(c, f, kappa),
                  "gdt_weighted_cost: dims must be positive multiples of kappa");
    GDT_CHECK_ARG(p >= 1.0 && batch >= 0, "gdt_weighted_cost: p must be >= 1");
    GDT_CHECK_ARG(mode == GDT_MODE_EXACT || mode == GDT_MODE_FAST, "gdt_weighted_cost: bad mode");
    int64_t need_sq = 0;
    for (int a = 0; a < ndim; ++a) need_sq += (dims[a] - 1) * (dims[a] - 1);
    GDT_CHECK_ARG(p == 1.0 || p == 2.0 || (cost_table != nullptr && max_sq >= need_sq),
                  "gdt_weighted_cost: cost_table required for p not in {1, 2}");
    if (batch == 0) return GDT_OK;
    cudaStream_t st = as_stream(stream);
    const int m = (int)ipow(kappa, ndim);
    const int64_t n = c.cells;
    if (mode == GDT_MODE_FAST && p == 2.0) {
        const int W = ndim + 1;
        double *mom = nullptr;
        if (malloc_async(reinterpret_cast<void **>(&mom), sizeof(double) * 2 * batch * n * W, st) != cudaSuccess)
            return cuda_status("gdt_weighted_cost: workspace");
        auto mk = [&](auto kern) {
            kern<<<grid_size(batch * n, 64), 64, 0, st>>>(mu, mom, batch, f, c, kappa);
            kern<<<grid_size(batch * n, 64), 64, 0, st>>>(nu, mom + batch * n * W, batch, f, c, kappa);
        };
        if (ndim == 2 && kappa == 4) mk(moments_kernel<2, 4>);
        else if (ndim == 2 && kappa == 8) mk(moments_kernel<2, 8>);
        else if (ndim == 2 && kappa == 2) mk(moments_kernel<2, 2>);
        else if (ndim == 3 && kappa == 4) mk(moments_kernel<3, 4>);
        else if (ndim == 3 && kappa == 2) mk(moments_kernel<3, 2>);
        else if (ndim == 1 && kappa == 4) mk(moments_kernel<1, 4>);
        else mk(moments_kernel<0, 0>);
        dim3 mg((unsigned)((n + 1023) / 1024), (unsigned)((n + MB_K - 1) / MB_K), (unsigned)batch);
        auto launch = [&](auto kern) {
            kern<<<mg, 256, 0, st>>>(mu_c, nu_c, mom, mom + batch * n * W, centre_cost, out, unused,
                                     c, kappa);
        };
        if (ndim == 1) launch(cbar_moments_kernel<1>);
        else if (ndim == 2) launch(cbar_moments_kernel<2>);
        else if (ndim == 3) launch(cbar_moments_kernel<3>);
        else launch(cbar_moments_kernel<4>);
        cudaFreeAsync(mom, st);
        return cuda_status("gdt_weighted_cost(moments)");
    }
    if (mode == GDT_MODE_FAST) {
        if (cbar_fast_diag(mu, nu, mu_c, nu_c, centre_cost, cost_table, max_sq, out, unused, batch,
                           f, c, kappa, p, st) == GDT_OK)
            return cuda_status("gdt_weighted_cost(diag)");
        const int rc = cbar_fast_toeplitz(mu, nu, mu_c, nu_c, centre_cost, cost_table, max_sq, out,
                                          unused, batch, f, c, kappa, p, st);
        if (rc == GDT_OK) return cuda_status("gdt_weighted_cost(toeplitz)");
        // outside the fp32 kernel's envelope: fall through to the exact fp64 kernel
    }
    if (ndim == 2 && (kappa == 2 || kappa == 4 || kappa == 8) && f.n[0] * kappa <= CE_CELLS &&
        (p == 1.0 || p == 2.0 || cost_table != nullptr)) {
        // exact order, 2-D: one row block per CTA, target cells in fine-row
        // order, costs from a 2-D table (cbar_exact2d_kernel)
        const int W = (int)std::max(f.n[0], f.n[1]);
        double *t2 = nullptr;
        if (malloc_async(reinterpret_cast<void **>(&t2), sizeof(double) * W * W, st) != cudaSuccess)
            return cuda_status("gdt_weighted_cost: workspace");
        cost2d_kernel<<<grid_size((int64_t)W * W, 256), 256, 0, st>>>(
            p == 2.0 ? nullptr : cost_table, p, W, W, t2);
        const int BR = (int)std::max<int64_t>(1, CE_CELLS / (f.n[0] * kappa));
        const int brows = (int)((c.n[1] + BR - 1) / BR);
        const size_t sb = sizeof(double) * (size_t)BR * c.n[0] * m;
        dim3 grid((unsigned)n, (unsigned)brows, (unsigned)batch);
        auto go = [&](auto kern) {
            if (sb > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
            kern<<<grid, CE_THREADS, sb, st>>>(mu, nu, mu_c, nu_c, centre_cost, t2, W, out,
                                               unused, f, c, BR);
        };
        if (kappa == 2) go(cbar_exact2d_kernel<2>);
        else if (kappa == 4) go(cbar_exact2d_kernel<4>);
        else go(cbar_exact2d_kernel<8>);
        cudaFreeAsync(t2, st);
        return cuda_status("gdt_weighted_cost(exact 2-D)");
    }
    if ((ndim == 2 || ndim == 3) && (kappa == 2 || kappa == 4 || kappa == 8) && m <= CE_CELLS &&
        (p == 1.0 || p == 2.0 || cost_table != nullptr)) {
        // exact order, one row block per CTA (cbar_exact_kernel)
        const int LT = (int)std::min<int64_t>(n, CE_CELLS / m);
        const size_t sb = sizeof(double) * LT * m;
        dim3 grid((unsigned)n, (unsigned)((n + LT - 1) / LT), (unsigned)batch);
        auto go = [&](auto kern) {
            if (sb > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
            // p in {1, 2} without a table: IEEE sqrt of / the integer squared distance
            kern<<<grid, CE_THREADS, sb, st>>>(mu, nu, mu_c, nu_c, centre_cost,
                                               p == 2.0 ? nullptr : cost_table, p, out, unused, f,
                                               c, LT);
        };
        if (ndim == 2) {
            if (kappa == 2) go(cbar_exact_kernel<2, 2>);
            else if (kappa == 4) go(cbar_exact_kernel<4, 2>);
            else go(cbar_exact_kernel<8, 2>);
        } else {
            if (kappa == 2) go(cbar_exact_kernel<2, 3>);
            else if (kappa == 4) go(cbar_exact_kernel<4, 3>);
            else go(cbar_exact_kernel<8, 3>);
        }
        return cuda_status("gdt_weighted_cost(exact)");
    }
    // tile shape: ~256 columns per CTA, KT row blocks per CTA
    int LT = m >= 256 ? 1 : 256 / m;
    if (LT > n) LT = (int)n;
    const int KT = 8;
    const int cols = LT * m;
    size_t sbytes = ((KT * cols * sizeof(double) + 7) / 8) * 8 + sizeof(double) * KT * m +
                    sizeof(int) * m * GDT_MAX_DIM;
    GDT_CHECK_ARG(sbytes <= 200 * 1024, "gdt_weighted_cost: kappa^d too large for this build");
    dim3 grid((unsigned)((n + LT - 1) / LT), (unsigned)((n + KT - 1) / KT), (unsigned)batch);
    if (sbytes > 48 * 1024)
        cudaFuncSetAttribute(cbar_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sbytes);
    cbar_tile_kernel<true><<<grid, 256, sbytes, st>>>(mu, nu, mu_c, nu_c, centre_cost, cost_table,
                                                      out, unused, f, c, kappa, m, p, KT, LT);
    return cuda_status("gdt_weighted_cost");
}

// ---------------------------------------------------------------------------
// C-bar of a coarser level from the C-bar of a finer one (nested blocks).
//
// With kappa_c = factor * kappa_f every coarse block K is the union of
// factor^d fine-level blocks k, and the numerator of C-bar (costs.py:128-171)
// is additive over them:
//   sum_{x in X_K, y in Y_L} C mu_x nu_y = sum_{k in K, l in L} C-bar_kl mu~_k nu~_l,
// so C-bar at kappa_c follows from C-bar at kappa_f in O(n_f^2) instead of a
// second O(N^2) pass over the fine cells.  One thread per (K, L): the
// children in ascending fine-coarse order (fixed: deterministic), fp64.
// Entries with mu~_K nu~_L == 0 take the centre cost, as in gdt_weighted_cost.
// ---------------------------------------------------------------------------
namespace gdt {

template <int ND>
__global__ void __launch_bounds__(256) cbar_pool_kernel(
    const double *__restrict__ cf, const double *__restrict__ mu_cf,
    const double *__restrict__ nu_cf, const double *__restrict__ mu_c,
    const double *__restrict__ nu_c, const double *__restrict__ centre,
    double *__restrict__ out, uint8_t *__restrict__ unused, int64_t batch, Grid gf, Grid gc,
    int factor) {
    // grid: x = (pair, coarse row K), y * blockDim + thread = coarse column L
    // (32-bit index arithmetic; consecutive threads read adjacent children)
    __shared__ int koff[64];    // flat fine-coarse offsets of the children of a block
    __shared__ double mks[64];  // mu~ of the children of K
    const int n = (int)gc.cells, nf = (int)gf.cells;
    const int kids = (int)ipow(factor, ND);
    const int64_t b = blockIdx.x / n;
    const int K = (int)(blockIdx.x - b * n);
    int cn[ND], fs[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) {
        cn[a] = (int)gc.n[a];
        fs[a] = (int)gf.stride[a];
    }
    int ko = 0;
    {
        int kk = K;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
            ko += (kk % cn[a]) * factor * fs[a];
            kk /= cn[a];
        }
    }
    for (int ci = threadIdx.x; ci < kids; ci += blockDim.x) {
        int off = 0, rem = ci;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
            off += (rem % factor) * fs[a];
            rem /= factor;
        }
        koff[ci] = off;
        mks[ci] = mu_cf[b * nf + ko + off];
    }
    __syncthreads();
    const int L = blockIdx.y * blockDim.x + threadIdx.x;
    if (L >= n) return;
    int lo = 0;
    {
        int ll = L;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
            lo += (ll % cn[a]) * factor * fs[a];
            ll /= cn[a];
        }
    }
    const double *cb = cf + b * (int64_t)nf * nf;
    const double *vf = nu_cf + b * nf + lo;
    double acc = 0.0;
    for (int ci = 0; ci < kids; ++ci) {
        const double mk = mks[ci];
        if (mk == 0.0) continue;  // weight zero: the entry is the centre cost, unused
        const double *row = cb + (int64_t)(ko + koff[ci]) * nf + lo;
        for (int cj = 0; cj < kids; ++cj) {
            const int o = koff[cj];
            acc += __ldg(row + o) * (mk * __ldg(vf + o));
        }
    }
    const int64_t idx = (b * n + K) * (int64_t)n + L;
    const double den = __dmul_rn(mu_c[b * n + K], nu_c[b * n + L]);
    const bool un = den == 0.0;
    out[idx] = un ? centre[(int64_t)K * n + L] : acc / den;
    if (unused) unused[idx] = un ? 1 : 0;
}

}  // namespace gdt

extern "C" int gdt_weighted_cost_pool(const double *cbar_fine, const double *mu_cf,
                                      const double *nu_cf, const double *mu_c,
                                      const double *nu_c, const double *centre_cost,
                                      double *out, uint8_t *unused, int64_t batch, int ndim,
                                      const int64_t *cdims_fine, int factor, void *stream) {
    Grid gf, gc;
    GDT_CHECK_ARG(factor >= 2 && make_grid(gf, ndim, cdims_fine) && make_coarse(gc, gf, factor),
                  "gdt_weighted_cost_pool: fine-level coarse dims must be positive multiples of factor");
    GDT_CHECK_ARG(batch >= 0 && cbar_fine && mu_cf && nu_cf && mu_c && nu_c && centre_cost && out,
                  "gdt_weighted_cost_pool: null argument");
    if (batch == 0) return GDT_OK;
    cudaStream_t st = as_stream(stream);
    GDT_CHECK_ARG(ipow(factor, ndim) <= 64 && gf.cells < (1ll << 31) &&
                      batch * gc.cells < (1ll << 31),
                  "gdt_weighted_cost_pool: factor^ndim must be <= 64, grids below 2^31 blocks");
    const int thr = gc.cells >= 256 ? 256 : (int)((gc.cells + 31) / 32 * 32);
    const dim3 grid((unsigned)(batch * gc.cells), (unsigned)((gc.cells + thr - 1) / thr));
    GDT_CHECK_ARG(grid.y <= 65535u, "gdt_weighted_cost_pool: coarse grid too large");
    auto go = [&](auto kern) {
        kern<<<grid, thr, 0, st>>>(cbar_fine, mu_cf, nu_cf, mu_c, nu_c, centre_cost, out, unused,
                                   batch, gf, gc, factor);
    };
    if (ndim == 1) go(cbar_pool_kernel<1>);
    else if (ndim == 2) go(cbar_pool_kernel<2>);
    else if (ndim == 3) go(cbar_pool_kernel<3>);
    else go(cbar_pool_kernel<4>);
    return cuda_status("gdt_weighted_cost_pool");
}
