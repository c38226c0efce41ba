// K2 fast mode, p != 2: diagonal register tiles + packed FFMA2.
//
//   numer_kl = sum_{c in Y_l} nu_c * G_kc,   G_kc = sum_{r in X_k} mu_r C(x_r - y_c)
//
// Observation: the cost of (row cell x = kappa*(k+j) + t, column c + j*kappa)
// does not depend on j.  A thread therefore owns a DIAGONAL tile -- for each of
// KR consecutive row blocks k+j along axis 0, the R consecutive columns
// c0 + j*kappa + r -- and one (source row, target row) pair needs only
// NCD = kappa + R - 1 distinct costs for KR*kappa*R FMAs.  Blocks j, j+1 are
// paired in the two lanes of sm_100's packed FFMA2 (fma.rn.f32x2), the cost
// entering as the broadcast scalar operand, so one instruction performs two
// FMAs.
//
// Each thread also owns TR consecutive target rows (axis 1).  The cost row of
// (source row sy, target row y0 + t) depends on sy - y0 - t only, so while the
// source rows of a block are visited in order a window of TR cost rows slides:
// one new row (NCD costs) per source row serves TR*KR*kappa*R FMAs.  p == 1
// costs come from sqrt.approx on the MUFU pipe; other p read an L1-resident
// fp32 table.  With everything in registers (<= 112 per thread, 2 CTAs/SM)
// the inner loop is FFMA2 + one MUFU row per source row + shared mu loads.
//
// Lane mapping: the G/TR lanes that hold the G higher-axis rows of one coarse
// block-row are consecutive (G/TR divides 32), so after the FMA loop the TR
// rows are folded in-thread and a butterfly over those lanes completes
// numer_kl for every (k+j, l) the group covers; the group leader stages it in
// shared memory and the CTA writes C-bar rows coalesced.  Every (k, l) is
// produced by exactly one lane group: no atomics, deterministic.
// Column windows start OFF cells left of the grid so every (block, column)
// pair is covered exactly once; out-of-grid columns are computed and dropped.
// Accuracy: fp32 FMA chains of kappa^d <= 64 terms (<= 3.8e-6 relative),
// fp32 folds, fp64 quotient; the fp32-mode contract of BASELINE.json is 1e-5
// on the bounds.
#include <algorithm>

#include "common.cuh"

namespace gdt {

constexpr int DG_MAX_THREADS = 128;  // 4 CTAs/SM at <= 128 registers

__device__ __forceinline__ unsigned long long dg_pack(float a, float b) {
    return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}

__device__ __forceinline__ float dg_sqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void dg_fma2(unsigned long long &acc, unsigned long long m2, float c) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(m2), "l"(dg_pack(c, c)));
}

// staged nu row length: N0 + 2 OFF, rounded to 4 (mod 32) floats against bank conflicts
__host__ __device__ __forceinline__ int dg_row_len(int n0, int off) {
    const int l = n0 + 2 * off;
    return ((l + 31) / 32) * 32 + 4;
}

// PER consecutive floats, vectorised (the start is a multiple of PER)
template <int PER>
__device__ __forceinline__ void dg_load(float *v, const float *src) {
    if constexpr (PER % 4 == 0) {
#pragma unroll
        for (int q = 0; q < PER / 4; ++q) {
            const float4 t = __ldg(reinterpret_cast<const float4 *>(src) + q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < PER / 2; ++q) {
            const float2 t = __ldg(reinterpret_cast<const float2 *>(src) + q);
            v[2 * q] = t.x; v[2 * q + 1] = t.y;
        }
    }
}

template <int KAPPA, int R>
struct DgCost {
    static constexpr int NCD = KAPPA + R - 1;
};

// one cost row: dx = base_dx + q (q < NCD), squared higher-axis offset hsq,
// axis-1 offset dy (table path of 2-D grids)
template <int NCD, int ND, bool P1>
__device__ __forceinline__ void dg_cost_row(float (&cw)[NCD], int base_dx, int hsq, int dy,
                                            const float *__restrict__ tab, int tab_max, int N0) {
    if constexpr (P1) {
        const float hf = (float)hsq, bx = (float)base_dx;
#pragma unroll
        for (int q = 0; q < NCD; ++q) {
            const float dx = bx + (float)q;
            cw[q] = dg_sqrt(__fmaf_rn(dx, dx, hf));
        }
    } else if constexpr (ND == 2) {
        const float *row = tab + (dy < 0 ? -dy : dy) * N0;
#pragma unroll
        for (int q = 0; q < NCD; ++q) {
            int dx = base_dx + q;
            dx = dx < 0 ? -dx : dx;
            cw[q] = __ldg(row + (dx < N0 ? dx : N0 - 1));  // clamp: dropped columns
        }
    } else {
#pragma unroll
        for (int q = 0; q < NCD; ++q) {
            const int dx = base_dx + q;
            const int sq = hsq + dx * dx;
            cw[q] = __ldg(tab + (sq < tab_max ? sq : tab_max));
        }
    }
}

template <int KAPPA, int KR, int TR, int R, int ND, bool P1>
__global__ void __launch_bounds__(DG_MAX_THREADS, 4) cbar_diag_kernel(
    const double *__restrict__ mu, const double *__restrict__ mu_c, const double *__restrict__ nu_c,
    const double *__restrict__ Ccentre, const float *__restrict__ tab, int tab_max,
    double *__restrict__ out, uint8_t *__restrict__ unused, Grid f, Grid c,
    const float *__restrict__ nup, const double *__restrict__ rmu, const double *__restrict__ rnu) {
    static_assert(KR % 2 == 0 && KAPPA % 2 == 0, "blocks and nu pairs fill FFMA2 lanes");
    static_assert(ND == 1 ? TR == 1 : KAPPA % TR == 0, "target rows of a thread share axis 2");
    extern __shared__ unsigned long long mus2[];  // [(th*KP + jp)*KAPPA + tx], then numer
    constexpr int NCD = DgCost<KAPPA, R>::NCD;
    constexpr int OFF = (((KR - 1) * KAPPA + R - 1) / R) * R;
    constexpr int G = ND == 1 ? 1 : (ND == 2 ? KAPPA : KAPPA * KAPPA);  // rows per block-row
    constexpr int LPB = G / TR;                                            // lanes per block-row
    constexpr int KP = KR / 2;
    constexpr int PER = KAPPA < R ? KAPPA : R;  // columns of one block inside a window
    constexpr int SY = ND == 1 ? 1 : KAPPA;     // source rows per axis-2 slice
    constexpr int SZ = G / SY;                  // axis-2 slices of a source block-row
    const int n = (int)c.cells, N0 = (int)f.n[0], n0 = (int)c.n[0];
    const int64_t N = f.cells;
    const int nthreads = blockDim.x;
    float *snum = reinterpret_cast<float *>(mus2 + G * KP * KAPPA);  // [KR][n] block numerators
    // nu rows in fp32 with OFF zero cells either side, prepared once per call
    // by dg_nu_pad_kernel: [B][fine rows][NL]
    const int NL = dg_row_len(N0, OFF);
    const int frows = (int)(N / N0);

    const int64_t b = blockIdx.y;
    const int tiles_x = (n0 + KR - 1) / KR;
    const int kt = blockIdx.x;
    const int k_hi = kt / tiles_x;
    const int kx0 = (kt - k_hi * tiles_x) * KR;
    const int kr_valid = n0 - kx0 < KR ? n0 - kx0 : KR;
    const double *mub = mu + b * N;

    int khc[GDT_MAX_DIM] = {0, 0, 0, 0};
    {
        int rem = k_hi;
#pragma unroll
        for (int a = 1; a < ND; ++a) {
            khc[a] = rem % (int)c.n[a];
            rem /= (int)c.n[a];
        }
    }
    for (int i = threadIdx.x; i < G * KP * KAPPA; i += nthreads) {
        const int th = i / (KP * KAPPA), rest = i - th * KP * KAPPA;
        const int jp = rest / KAPPA, tx = rest - jp * KAPPA;
        int64_t hoff = 0;
        int rem = th;
#pragma unroll
        for (int a = 1; a < ND; ++a) {
            const int ta = rem % KAPPA;
            rem /= KAPPA;
            hoff += (int64_t)(khc[a] * KAPPA + ta) * f.stride[a];
        }
        float v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * jp + h;
            v[h] = j < kr_valid ? (float)mub[hoff + (kx0 + j) * KAPPA + tx] : 0.f;
        }
        mus2[i] = dg_pack(v[0], v[1]);
    }
    __syncthreads();

    // work units (block-row lb, column segment seg, row group u), u fastest;
    // consecutive threads take consecutive units, whole idle warps leave early
    const int segs = (N0 + OFF) / R;
    const int n_hi = n / n0;  // coarse block-rows
    const int units = n_hi * segs * LPB;
    const int warp0 = threadIdx.x & ~31;
    const int numer_row = n;  // snum row stride

    // unit decomposition advanced incrementally (no divisions per pass): the
    // row group u is fixed (LPB divides the 32-aligned CTA size), seg and lb
    // step by the CTA size in mixed radix (segs, n_hi)
    const int u = threadIdx.x % LPB;
    const int dq = nthreads / LPB, dseg = dq % segs, dlb = dq / segs;
    int seg = (threadIdx.x / LPB) % segs, lb = threadIdx.x / (LPB * segs);
    int rstride[GDT_MAX_DIM] = {0, 0, 0, 0};  // fine-row stride of each higher axis
#pragma unroll
    for (int a = 1; a < ND; ++a) rstride[a] = (int)(f.stride[a] / N0);
    for (int w0 = 0; w0 + warp0 < units; w0 += nthreads) {
        const bool active = w0 + (int)threadIdx.x < units;
        if (w0 > 0) {
            seg += dseg;
            lb += dlb;
            if (seg >= segs) {
                seg -= segs;
                ++lb;
            }
        }
        const int lbe = active ? lb : 0;  // coarse block-row (flat over the higher axes)
        const int c0 = seg * R - OFF;
        const int base_dx = kx0 * KAPPA - c0 - (R - 1);
        int chc[GDT_MAX_DIM] = {0, 0, 0, 0};  // fine higher coordinates of this lane's first row
        int rowid = 0;                         // fine row (flat over the higher axes) of it
        {
            int rem = lbe, rr = u * TR;
#pragma unroll
            for (int a = 1; a < ND; ++a) {
                int la = rem;
                if (a < ND - 1) {
                    la = rem % (int)c.n[a];
                    rem /= (int)c.n[a];
                }
                chc[a] = la * KAPPA + rr % KAPPA;
                rr /= KAPPA;
                rowid += chc[a] * rstride[a];
            }
        }
        unsigned long long acc[TR][KP][R];
#pragma unroll
        for (int t = 0; t < TR; ++t)
#pragma unroll
            for (int jp = 0; jp < KP; ++jp)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[t][jp][r] = 0ull;
        if (active) {
            // axis-1 offset of (source row 0, target row y0); axis-2 offset per slice
            const int dy0 = ND >= 2 ? khc[1] * KAPPA - chc[1] : 0;
#pragma unroll 1
            for (int sz = 0; sz < SZ; ++sz) {
                int hz = 0;
                if constexpr (ND == 3) {
                    const int dz = khc[2] * KAPPA + sz - chc[2];
                    hz = dz * dz;
                }
                // cw[t] = cost row of (source row sy, target row y0 + t): dy = dy0 + sy - t
                float cw[TR][NCD];
#pragma unroll
                for (int t = 1; t < TR; ++t) {
                    const int dy = dy0 - t;
                    dg_cost_row<NCD, ND, P1>(cw[t], base_dx, dy * dy + hz, dy, tab, tab_max, N0);
                }
#pragma unroll
                for (int sy = 0; sy < SY; ++sy) {
                    if (sy > 0) {  // slide the window (register renames once unrolled)
#pragma unroll
                        for (int t = TR - 1; t >= 1; --t)
#pragma unroll
                            for (int q = 0; q < NCD; ++q) cw[t][q] = cw[t - 1][q];
                    }
                    {
                        const int dy = dy0 + sy;
                        dg_cost_row<NCD, ND, P1>(cw[0], base_dx, dy * dy + hz, dy, tab, tab_max,
                                                 N0);
                    }
                    const unsigned long long *mrow = mus2 + (sz * SY + sy) * KP * KAPPA;
#pragma unroll
                    for (int jp = 0; jp < KP; ++jp) {
#pragma unroll
                        for (int tx = 0; tx < KAPPA; ++tx) {
                            const unsigned long long m2 = mrow[jp * KAPPA + tx];
#pragma unroll
                            for (int t = 0; t < TR; ++t)
#pragma unroll
                                for (int r = 0; r < R; ++r)
                                    dg_fma2(acc[t][jp][r], m2, cw[t][tx - r + R - 1]);
                        }
                    }
                }
            }
        }
        // fold: the TR rows in-thread, then the G/TR lanes of the block-row;
        // the leader stages numer_kl for every (k+j, l) the group covers
        const float *nrow = nup + ((int64_t)b * frows + rowid) * NL + OFF + c0;
        // target block of window column 0 (c0 is a multiple of kappa) and its staging slot
        const int lc0 = c0 / KAPPA;
        float *srow = snum + lbe * n0 + lc0;
        const bool leader = u == 0 && active;
#pragma unroll
        for (int jp = 0; jp < KP; ++jp) {
#pragma unroll
            for (int g = 0; g < R / PER; ++g) {
                // blocks 2jp, 2jp+1 (the two lanes of acc): s = sum_t,r acc * nu
                const int oA = 2 * jp * KAPPA + g * PER;  // window offset of block 2jp's columns
                // scalar FMAs on the two halves of each accumulator pair (no repacking of nu)
                float sv[2] = {0.f, 0.f};
#pragma unroll
                for (int t = 0; t < TR; ++t) {
                    float nvA[PER], nvB[PER];
                    dg_load<PER>(nvA, nrow + t * NL + oA);
                    dg_load<PER>(nvB, nrow + t * NL + oA + KAPPA);
#pragma unroll
                    for (int r = 0; r < PER; ++r) {
                        const unsigned long long a2 = acc[t][jp][g * PER + r];
                        sv[0] = __fmaf_rn(__uint_as_float((unsigned)(a2 & 0xffffffffu)), nvA[r], sv[0]);
                        sv[1] = __fmaf_rn(__uint_as_float((unsigned)(a2 >> 32)), nvB[r], sv[1]);
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 2 * jp + h;
                    const int bo = (oA + h * KAPPA) / KAPPA;  // target block offset in the window
                    float sh = sv[h];
#pragma unroll
                    for (int o = 1; o < LPB; o <<= 1) sh += __shfl_xor_sync(0xffffffffu, sh, o, LPB);
                    const unsigned lc = (unsigned)(lc0 + bo);
                    if (leader && lc < (unsigned)n0 && j < kr_valid)
                        srow[j * numer_row + bo] = sh;  // unique writer per entry
                }
            }
        }
    }
    __syncthreads();
    // coalesced row writes of C-bar = numer / (mu~ nu~) (centre cost where 0);
    // fp32-mode quotient through precomputed reciprocals (~2 ulp of fp64)
    const int64_t kbase = (int64_t)b * n + k_hi * n0 + kx0;
    if (n & 1) {
        for (int i = threadIdx.x; i < kr_valid * n; i += nthreads) {
            const int j = i / n, l = i - j * n;
            const int64_t kb = kbase + j, oi = kb * n + l;
            const bool un = __dmul_rn(mu_c[kb], nu_c[b * n + l]) == 0.0;
            out[oi] = un ? Ccentre[(kb - b * n) * n + l] : (double)snum[i] * rmu[kb] * rnu[b * n + l];
            if (unused) unused[oi] = un ? 1 : 0;
        }
    } else {  // row by row, two consecutive l per thread
        const double *nub_c = nu_c + b * n, *rnub = rnu + b * n;
        for (int j = 0; j < kr_valid; ++j) {
            const int64_t kb = kbase + j;
            const double mk = mu_c[kb], rk = rmu[kb];
            const float *sj = snum + j * n;
            double *oj = out + kb * n;
            uint8_t *uj = unused ? unused + kb * n : nullptr;
            const double *cj = Ccentre + (kb - (int64_t)b * n) * n;
            for (int l = 2 * threadIdx.x; l < n; l += 2 * nthreads) {
                const double2 nl = *reinterpret_cast<const double2 *>(nub_c + l);
                const double2 rl = *reinterpret_cast<const double2 *>(rnub + l);
                const float2 sn = *reinterpret_cast<const float2 *>(sj + l);
                const bool u0 = __dmul_rn(mk, nl.x) == 0.0, u1 = __dmul_rn(mk, nl.y) == 0.0;
                double2 o;
                o.x = u0 ? cj[l] : (double)sn.x * rk * rl.x;
                o.y = u1 ? cj[l + 1] : (double)sn.y * rk * rl.y;
                *reinterpret_cast<double2 *>(oj + l) = o;
                if (uj) *reinterpret_cast<uchar2 *>(uj + l) = make_uchar2(u0 ? 1 : 0, u1 ? 1 : 0);
            }
        }
    }
}

// nu as padded fp32 rows [B][rows][NL] (OFF zeros either side) and the
// reciprocals of the coarse masses (0 where the mass is 0)
__global__ void dg_nu_pad_kernel(const double *__restrict__ nu, float *__restrict__ nup,
                                 int64_t batch, int64_t rows, int N0, int NL, int OFF) {
    const int64_t total = batch * rows * NL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / NL;
        const int x = (int)(i - r * NL) - OFF;
        nup[i] = x >= 0 && x < N0 ? (float)nu[r * N0 + x] : 0.f;
    }
}

__global__ void dg_recip_kernel(const double *__restrict__ a, double *__restrict__ r, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        r[i] = a[i] > 0.0 ? 1.0 / a[i] : 0.0;
}

__global__ void dg_table2d_kernel(const double *__restrict__ g, float *__restrict__ t, int64_t ny,
                                  int64_t nx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ny * nx;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t dy = i / nx, dx = i - dy * nx;
        t[i] = (float)g[dx * dx + dy * dy];
    }
}

__global__ void dg_table1d_kernel(const double *__restrict__ g, float *__restrict__ t, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        t[i] = (float)g[i];
}

template <int KAPPA, int KR, int TR, int R>
static int dg_launch(const double *mu, const double *nu, const double *mu_c, const double *nu_c,
                     const double *Ccentre, const double *table, int64_t max_sq, double *out,
                     uint8_t *unused, int64_t batch, const Grid &f, const Grid &c, bool p1,
                     cudaStream_t st) {
    constexpr int OFF = (((KR - 1) * KAPPA + R - 1) / R) * R;
    const int Gr = (int)ipow(KAPPA, f.nd - 1);
    const int tr = f.nd == 1 ? 1 : TR;
    const int lpb = Gr / tr;  // lanes per block-row
    if (lpb > 32 || f.n[0] % R || f.cells >= (1ll << 31)) return GDT_ERR_UNSUPPORTED;
    const int segs = (int)((f.n[0] + OFF) / R);
    const int64_t units = (c.cells / c.n[0]) * segs * lpb;
    const int threads = (int)std::min<int64_t>(DG_MAX_THREADS, (units + 31) / 32 * 32);
    const int64_t n = c.cells;
    const size_t bytes = sizeof(unsigned long long) * Gr * (KR / 2) * KAPPA +
                         sizeof(float) * ((KR * n + 3) & ~3);
    if (bytes > 56 * 1024) return GDT_ERR_UNSUPPORTED;
    float *ftab = nullptr;
    int tab_max = 0;
    if (!p1) {
        const bool two_d = f.nd == 2;
        const int64_t cnt = two_d ? f.n[0] * f.n[1] : max_sq + 1;
        if (malloc_async(reinterpret_cast<void **>(&ftab), sizeof(float) * cnt, st) != cudaSuccess) return GDT_ERR_CUDA;
        if (two_d) dg_table2d_kernel<<<grid_size(cnt, 256), 256, 0, st>>>(table, ftab, f.n[1], f.n[0]);
        else dg_table1d_kernel<<<grid_size(cnt, 256), 256, 0, st>>>(table, ftab, cnt);
        tab_max = (int)max_sq;
    }
    const int NL = dg_row_len((int)f.n[0], OFF);
    const int64_t frows = f.cells / f.n[0];
    float *nup = nullptr;
    double *rmu = nullptr, *rnu = nullptr;
    if (malloc_async(reinterpret_cast<void **>(&nup), sizeof(float) * batch * frows * NL, st) !=
            cudaSuccess ||
        malloc_async(reinterpret_cast<void **>(&rmu), sizeof(double) * 2 * batch * n, st) !=
            cudaSuccess) {
        if (ftab) cudaFreeAsync(ftab, st);
        return GDT_ERR_CUDA;
    }
    rnu = rmu + batch * n;
    dg_nu_pad_kernel<<<grid_size(batch * frows * NL, 256), 256, 0, st>>>(nu, nup, batch, frows,
                                                                         (int)f.n[0], NL, OFF);
    dg_recip_kernel<<<grid_size(batch * n, 256), 256, 0, st>>>(mu_c, rmu, batch * n);
    dg_recip_kernel<<<grid_size(batch * n, 256), 256, 0, st>>>(nu_c, rnu, batch * n);
    const int64_t tiles_x = (c.n[0] + KR - 1) / KR;
    dim3 grid((unsigned)(tiles_x * (n / c.n[0])), (unsigned)batch);
    auto run = [&](auto kern) {
        if (bytes > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        kern<<<grid, threads, bytes, st>>>(mu, mu_c, nu_c, Ccentre, ftab, tab_max, out, unused, f,
                                           c, nup, rmu, rnu);
    };
    switch (f.nd * 2 + (p1 ? 1 : 0)) {
        case 2: run(cbar_diag_kernel<KAPPA, KR, 1, R, 1, false>); break;
        case 3: run(cbar_diag_kernel<KAPPA, KR, 1, R, 1, true>); break;
        case 4: run(cbar_diag_kernel<KAPPA, KR, TR, R, 2, false>); break;
        case 5: run(cbar_diag_kernel<KAPPA, KR, TR, R, 2, true>); break;
        case 6: run(cbar_diag_kernel<KAPPA, KR, TR, R, 3, false>); break;
        case 7: run(cbar_diag_kernel<KAPPA, KR, TR, R, 3, true>); break;
        default: break;
    }
    if (ftab) cudaFreeAsync(ftab, st);
    cudaFreeAsync(nup, st);
    cudaFreeAsync(rmu, st);
    return GDT_OK;
}

int cbar_fast_diag(const double *mu, const double *nu, const double *mu_c, const double *nu_c,
                   const double *Ccentre, const double *table, int64_t max_sq, double *out,
                   uint8_t *unused, int64_t batch, const Grid &f, const Grid &c, int kappa, double p,
                   cudaStream_t st) {
    const bool p1 = p == 1.0;
    if ((!p1 && table == nullptr) || f.nd > 3 || ipow(kappa, f.nd) > 64) return GDT_ERR_UNSUPPORTED;
    // tile shape per kappa: (KR row blocks, TR target rows, R columns) per
    // thread, the fastest of the shapes measured on B200 (KR x TR x R with
    // 64 accumulator floats and no spills at 128 registers)
#define DG_ARGS mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused, batch, f, c, p1, st
    switch (kappa) {
        case 2: return dg_launch<2, 8, 1, 8>(DG_ARGS);
        case 4: return dg_launch<4, 4, 2, 8>(DG_ARGS);
        case 8: return dg_launch<8, 2, 2, 8>(DG_ARGS);
        default: return GDT_ERR_UNSUPPORTED;
    }
#undef DG_ARGS
}

}  // namespace gdt
