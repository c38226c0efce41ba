// K2 fast mode, p != 2: diagonal register tiles + packed FFMA2.
//
//   numer_kl = sum_{c in Y_l} nu_c * G_kc,   G_kc = sum_{r in X_k} mu_r C(x_r - y_c)
//
// Observation: the cost of (row cell x = kappa*(k+j) + t, column c + j*kappa)
// does not depend on j.  A thread therefore owns a DIAGONAL tile -- for each of
// KR consecutive row blocks k+j along axis 0, the R = 8 columns
// c0 + j*kappa + r -- and one higher-axis row offset needs only
// kappa + R - 1 distinct costs for KR*kappa*R FMAs.  Blocks j, j+1 are paired
// in the two lanes of sm_100's packed FFMA2 (fma.rn.f32x2), the cost entering
// as a broadcast scalar operand, so one instruction performs two FMAs.
// p == 1 costs come from sqrt.approx on the MUFU pipe (dx^2 fixed per thread,
// dy^2 per row offset); other p read an L1-resident fp32 table.  Column
// windows start OFF cells left of the grid so every (block, column) pair is
// covered exactly once; out-of-grid columns are computed and discarded.
// Accuracy: fp32 FMA chains of kappa^d <= 64 terms (<= 3.8e-6 relative), fp64
// block sums; fp32 mode contract of BASELINE.json is 1e-5.
#include "common.cuh"

namespace gdt {

constexpr int DG_THREADS = 256;
constexpr int DG_R = 8;

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

template <int KAPPA, int KR, int ND, bool P1>
__global__ void __launch_bounds__(DG_THREADS, 2) cbar_diag_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const double *__restrict__ mu_c,
    const double *__restrict__ nu_c, const double *__restrict__ Ccentre,
    const float *__restrict__ tab, int tab_max, double *__restrict__ out,
    uint8_t *__restrict__ unused, Grid f, Grid c) {
    static_assert(KR % 2 == 0, "blocks are paired in FFMA2 lanes");
    extern __shared__ double smem[];
    constexpr int R = DG_R;
    constexpr int NCD = KAPPA + R - 1;                      // distinct costs per row offset
    constexpr int OFF = (((KR - 1) * KAPPA + R - 1) / R) * R;  // left extension of the windows
    constexpr int m_hi = ND == 1 ? 1 : (ND == 2 ? KAPPA : KAPPA * KAPPA);
    constexpr int KP = KR / 2;
    constexpr int SPAN = (KR - 1) * KAPPA + R;              // columns touched by one thread
    const int n = (int)c.cells, N0 = (int)f.n[0], n0 = (int)c.n[0];
    const int64_t N = f.cells;

    double *numer = smem;                                                  // [KR][n]
    unsigned long long *mus2 = reinterpret_cast<unsigned long long *>(numer + KR * n);
    // mus2[(th * KP + jp) * KAPPA + tx] = (mu[k+2jp][t], mu[k+2jp+1][t])

    const int64_t b = blockIdx.y;
    const int tiles_x = (n0 + KR - 1) / KR;
    const int kt = blockIdx.x;
    const int k_hi = kt / tiles_x;
    const int kx0 = (kt - k_hi * tiles_x) * KR;
    const int kr_valid = n0 - kx0 < KR ? n0 - kx0 : KR;
    const double *mub = mu + b * N, *nub = nu + b * N;

    int khc[GDT_MAX_DIM] = {0, 0, 0, 0};
    {
        int rem = k_hi;
#pragma unroll
        for (int a = 1; a < ND; ++a) {
            khc[a] = rem % (int)c.n[a];
            rem /= (int)c.n[a];
        }
    }
    for (int i = threadIdx.x; i < m_hi * KP * KAPPA; i += DG_THREADS) {
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
    for (int i = threadIdx.x; i < KR * n; i += DG_THREADS) numer[i] = 0.0;
    __syncthreads();

    const int segs = (N0 + OFF) / R;
    const int rows_per_pass = DG_THREADS / segs;
    const int64_t H = N / N0;
    const int seg = threadIdx.x % segs, rloc = threadIdx.x / segs;
    const int c0 = seg * R - OFF;
    const int base_dx = kx0 * KAPPA - c0 - (R - 1);
    float dx2[NCD];
#pragma unroll
    for (int q = 0; q < NCD; ++q) {
        const float dx = (float)(base_dx + q);
        dx2[q] = dx * dx;
    }

    for (int64_t h0 = 0; h0 < H; h0 += rows_per_pass) {
        const int64_t hrow = h0 + rloc;
        if (rloc >= rows_per_pass || hrow >= H) continue;
        int chc[GDT_MAX_DIM] = {0, 0, 0, 0};
        {
            int64_t rem = hrow;
#pragma unroll
            for (int a = 1; a < ND; ++a) {
                chc[a] = (int)(rem % f.n[a]);
                rem /= f.n[a];
            }
        }
        unsigned long long acc[KP][R];
#pragma unroll
        for (int jp = 0; jp < KP; ++jp)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[jp][r] = 0ull;

#pragma unroll 1
        for (int th = 0; th < m_hi; ++th) {
            int rem = th, hsq = 0, dy1 = 0;
#pragma unroll
            for (int a = 1; a < ND; ++a) {
                const int ta = rem % KAPPA;
                rem /= KAPPA;
                const int d = khc[a] * KAPPA + ta - chc[a];
                if (a == 1) dy1 = d < 0 ? -d : d;
                hsq += d * d;
            }
            float cst[NCD];
            if (P1) {
                const float hf = (float)hsq;
#pragma unroll
                for (int q = 0; q < NCD; ++q) cst[q] = dg_sqrt(dx2[q] + hf);
            } else if (ND == 2) {
                const float *row = tab + dy1 * N0;
#pragma unroll
                for (int q = 0; q < NCD; ++q) {
                    int dx = base_dx + q;
                    dx = dx < 0 ? -dx : dx;
                    cst[q] = __ldg(row + (dx < N0 ? dx : N0 - 1));  // clamp: masked columns
                }
            } else {
#pragma unroll
                for (int q = 0; q < NCD; ++q) {
                    const int dx = base_dx + q;
                    const int sq = hsq + dx * dx;
                    cst[q] = __ldg(tab + (sq < tab_max ? sq : tab_max));
                }
            }
            const unsigned long long *mrow = mus2 + th * KP * KAPPA;
#pragma unroll
            for (int jp = 0; jp < KP; ++jp) {
#pragma unroll
                for (int tx = 0; tx < KAPPA; ++tx) {
                    const unsigned long long m2 = mrow[jp * KAPPA + tx];
#pragma unroll
                    for (int r = 0; r < R; ++r) dg_fma2(acc[jp][r], m2, cst[tx - r + R - 1]);
                }
            }
        }
        // fold: numer[j][l] += sum over the thread's columns of block l of nu_c * G
        const int64_t rowbase = hrow * N0;
        float nv[SPAN];
#pragma unroll
        for (int q = 0; q < SPAN; ++q) {
            const int col = c0 + q;
            nv[q] = (col >= 0 && col < N0) ? (float)nub[rowbase + col] : 0.f;
        }
        int l_hi = 0;
#pragma unroll
        for (int a = ND - 1; a >= 1; --a) l_hi = l_hi * (int)c.n[a] + chc[a] / KAPPA;
        constexpr int PER = KAPPA < R ? KAPPA : R;
#pragma unroll
        for (int jp = 0; jp < KP; ++jp) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = 2 * jp + h;
                if (j >= kr_valid) continue;
#pragma unroll
                for (int g = 0; g < R / PER; ++g) {
                    const int cs = c0 + j * KAPPA + g * PER;  // first column of the group
                    if (cs < 0 || cs >= N0) continue;
                    float s = 0.f;
#pragma unroll
                    for (int r = g * PER; r < (g + 1) * PER; ++r) {
                        const unsigned long long a2 = acc[jp][r];
                        const float gv = __uint_as_float((unsigned)(h ? (a2 >> 32) : (a2 & 0xffffffffu)));
                        s = fmaf(nv[j * KAPPA + r], gv, s);
                    }
                    atomicAdd(&numer[j * n + l_hi * n0 + cs / KAPPA], (double)s);
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kr_valid * n; i += DG_THREADS) {
        const int j = i / n, l = i - j * n;
        const int k = k_hi * n0 + kx0 + j;
        const double denom = __dmul_rn(mu_c[b * n + k], nu_c[b * n + l]);
        const int64_t oi = ((int64_t)b * n + k) * n + l;
        const bool un = denom == 0.0;
        out[oi] = un ? Ccentre[(int64_t)k * n + l] : numer[i] / denom;
        unused[oi] = un ? 1 : 0;
    }
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

template <int KAPPA, int KR>
static int dg_launch(const double *mu, const double *nu, const double *mu_c, const double *nu_c,
                     const double *Ccentre, const double *table, int64_t max_sq, double *out,
                     uint8_t *unused, int64_t batch, const Grid &f, const Grid &c, bool p1,
                     cudaStream_t st) {
    constexpr int OFF = (((KR - 1) * KAPPA + DG_R - 1) / DG_R) * DG_R;
    if (f.n[0] % DG_R || (f.n[0] + OFF) / DG_R > DG_THREADS) return GDT_ERR_UNSUPPORTED;
    if (f.cells >= (1ll << 31)) return GDT_ERR_UNSUPPORTED;
    const int64_t n = c.cells;
    int m_hi = 1;
    for (int a = 1; a < f.nd; ++a) m_hi *= KAPPA;
    const size_t bytes = sizeof(double) * KR * n + sizeof(unsigned long long) * m_hi * KR / 2 * KAPPA;
    if (bytes > 200 * 1024) return GDT_ERR_UNSUPPORTED;
    float *ftab = nullptr;
    int tab_max = 0;
    if (!p1) {
        const bool two_d = f.nd == 2;
        const int64_t cnt = two_d ? f.n[0] * f.n[1] : max_sq + 1;
        if (cudaMallocAsync(&ftab, sizeof(float) * cnt, st) != cudaSuccess) return GDT_ERR_CUDA;
        if (two_d) dg_table2d_kernel<<<grid_size(cnt, 256), 256, 0, st>>>(table, ftab, f.n[1], f.n[0]);
        else dg_table1d_kernel<<<grid_size(cnt, 256), 256, 0, st>>>(table, ftab, cnt);
        tab_max = (int)max_sq;
    }
    const int64_t tiles_x = (c.n[0] + KR - 1) / KR;
    dim3 grid((unsigned)(tiles_x * (n / c.n[0])), (unsigned)batch);
    auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        kern<<<grid, DG_THREADS, bytes, st>>>(mu, nu, mu_c, nu_c, Ccentre, ftab, tab_max, out,
                                              unused, f, c);
    };
    switch (f.nd * 2 + (p1 ? 1 : 0)) {
        case 2: run(cbar_diag_kernel<KAPPA, KR, 1, false>); break;
        case 3: run(cbar_diag_kernel<KAPPA, KR, 1, true>); break;
        case 4: run(cbar_diag_kernel<KAPPA, KR, 2, false>); break;
        case 5: run(cbar_diag_kernel<KAPPA, KR, 2, true>); break;
        case 6: run(cbar_diag_kernel<KAPPA, KR, 3, false>); break;
        case 7: run(cbar_diag_kernel<KAPPA, KR, 3, true>); break;
        default: break;
    }
    if (ftab) cudaFreeAsync(ftab, st);
    return GDT_OK;
}

int cbar_fast_diag(const double *mu, const double *nu, const double *mu_c, const double *nu_c,
                   const double *Ccentre, const double *table, int64_t max_sq, double *out,
                   uint8_t *unused, int64_t batch, const Grid &f, const Grid &c, int kappa, double p,
                   cudaStream_t st) {
    const bool p1 = p == 1.0;
    if ((!p1 && table == nullptr) || f.nd > 3 || ipow(kappa, f.nd) > 64) return GDT_ERR_UNSUPPORTED;
    switch (kappa) {
        case 2: return dg_launch<2, 8>(mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused,
                                       batch, f, c, p1, st);
        case 4: return dg_launch<4, 4>(mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused,
                                       batch, f, c, p1, st);
        case 8: return dg_launch<8, 2>(mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused,
                                       batch, f, c, p1, st);
        default: return GDT_ERR_UNSUPPORTED;
    }
}

}  // namespace gdt
