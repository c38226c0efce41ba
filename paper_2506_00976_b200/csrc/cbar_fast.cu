// K2 fast mode (fp32 mode of BASELINE.json), p != 2: register-tiled Toeplitz
// evaluation of
//   numer_kl = sum_{c in Y_l} nu_c * G_kc,   G_kc = sum_{r in X_k} mu_r rho(x_r, y_c)^p
// (costs.py:128-171 computes the same quantity in fp64; here G is accumulated
// in fp32 FFMA -- at most kappa^d <= 64 terms, so <= 64 ulp = 3.8e-6 worst-case
// relative error -- and the block sums in fp64.)
//
// A CTA owns KR consecutive row blocks along axis 0 (same higher block
// coordinates) and sweeps every column cell of its pair.  A thread owns R = 8
// consecutive columns along axis 0; for one higher-axis row offset of the
// blocks it needs only kappa*KR + R - 1 distinct costs (the cost depends on
// x_r - y_c only), which it reads from a shared-memory table, and performs
// kappa*KR*R FFMAs on them.  Column partial sums go to a per-CTA fp64
// shared-memory accumulator numer[KR][n] that is written out once.
#include "common.cuh"

namespace gdt {

constexpr int CF_THREADS = 256;
constexpr int CF_R = 8;


// float cost tables read through L1: [|dy|][|dx|] for d == 2, [sq] otherwise
__global__ void ftable2d_kernel(const double *__restrict__ g, float *__restrict__ t, int64_t ny,
                                int64_t nx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ny * nx;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t dy = i / nx, dx = i - dy * nx;
        t[i] = (float)g[dx * dx + dy * dy];
    }
}

__global__ void ftable1d_kernel(const double *__restrict__ g, float *__restrict__ t, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        t[i] = (float)g[i];
}

__device__ __forceinline__ float sqrt_apx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// P1: p == 1 costs are generated as sqrt.approx(dx^2 + dy^2) on the MUFU pipe
// (no table loads; dx^2 is fixed per pass, dy^2 per row offset)
template <int KAPPA, int KR, int ND, bool P1>
__global__ void __launch_bounds__(CF_THREADS, 2) cbar_toeplitz_kernel(
    const double *__restrict__ mu, const double *__restrict__ nu, const double *__restrict__ mu_c,
    const double *__restrict__ nu_c, const double *__restrict__ Ccentre,
    const float *__restrict__ tab, double *__restrict__ out, uint8_t *__restrict__ unused, Grid f,
    Grid c) {
    extern __shared__ double smem[];
    constexpr int M_X = KAPPA * KR;          // row cells along x in the tile
    constexpr int NC = M_X + CF_R - 1;       // distinct costs per hi-row offset
    const int64_t n = c.cells, N = f.cells, N0 = f.n[0], n0 = c.n[0];
    constexpr int nd = ND;
    constexpr int TAB2D = 0, TAB1D = 1;
    constexpr int TAB = ND == 2 ? TAB2D : TAB1D;
    constexpr int m_hi = ND == 1 ? 1 : (ND == 2 ? KAPPA : KAPPA * KAPPA);

    double *numer = smem;                                    // [KR][n]
    float *mus = reinterpret_cast<float *>(numer + KR * n);  // [m_hi][KR*KAPPA]

    const int64_t b = blockIdx.y;
    const int64_t tiles_x = (n0 + KR - 1) / KR;
    const int64_t kt = blockIdx.x;
    const int64_t k_hi = kt / tiles_x;          // flat index of the higher block coords
    const int64_t kx0 = (kt - k_hi * tiles_x) * KR;
    const int kr_valid = (int)(n0 - kx0 < KR ? n0 - kx0 : KR);
    const double *mub = mu + b * N, *nub = nu + b * N;

    // higher block coordinates of this tile
    int64_t khc[GDT_MAX_DIM] = {0, 0, 0, 0};
    {
        int64_t rem = k_hi;
#pragma unroll
        for (int a = 1; a < nd; ++a) {
            khc[a] = rem % c.n[a];
            rem /= c.n[a];
        }
    }

    // stage: mu of the KR blocks (float), zero accumulators
    for (int i = threadIdx.x; i < m_hi * M_X; i += CF_THREADS) {
        const int th = i / M_X, q = i - th * M_X;
        const int kk = q / KAPPA, tx = q - kk * KAPPA;
        float v = 0.f;
        if (kk < kr_valid) {
            int64_t off = (kx0 + kk) * KAPPA + tx;
            int rem = th;
#pragma unroll
            for (int a = 1; a < nd; ++a) {
                const int ta = rem % KAPPA;
                rem /= KAPPA;
                off += (khc[a] * KAPPA + ta) * f.stride[a];
            }
            v = (float)mub[off];
        }
        mus[i] = v;
    }
    for (int64_t i = threadIdx.x; i < KR * n; i += CF_THREADS) numer[i] = 0.0;
    __syncthreads();

    const int segs = (int)(N0 / CF_R);
    const int rows_per_pass = CF_THREADS / segs;
    const int64_t H = N / N0;  // higher-coordinate rows
    const int seg = threadIdx.x % segs, rloc = threadIdx.x / segs;
    const int64_t cx0 = (int64_t)seg * CF_R;
    const int64_t base_dx = kx0 * KAPPA - cx0 - (CF_R - 1);  // dx of cost slot q = base_dx + q

    for (int64_t h0 = 0; h0 < H; h0 += rows_per_pass) {
        const int64_t hrow = h0 + rloc;
        const bool active = rloc < rows_per_pass && hrow < H;
        float acc[KR][CF_R];
#pragma unroll
        for (int kk = 0; kk < KR; ++kk)
#pragma unroll
            for (int r = 0; r < CF_R; ++r) acc[kk][r] = 0.f;
        int64_t chc[GDT_MAX_DIM] = {0, 0, 0, 0};
        {
            int64_t rem = active ? hrow : 0;
#pragma unroll
            for (int a = 1; a < nd; ++a) {
                chc[a] = rem % f.n[a];
                rem /= f.n[a];
            }
        }
        float dx2[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const float dx = (float)(base_dx + q);
            dx2[q] = dx * dx;
        }
        if (active) {
#pragma unroll 1
            for (int th = 0; th < m_hi; ++th) {
                // higher-axis squared distance of this row offset
                int rem = th;
                int64_t hsq = 0, dy1 = 0;
#pragma unroll
                for (int a = 1; a < nd; ++a) {
                    const int ta = rem % KAPPA;
                    rem /= KAPPA;
                    const int64_t d = khc[a] * KAPPA + ta - chc[a];
                    if (a == 1) dy1 = d < 0 ? -d : d;
                    hsq += d * d;
                }
                float cst[NC];
                if (P1) {
                    const float hsqf = (float)hsq;
#pragma unroll
                    for (int q = 0; q < NC; ++q) cst[q] = sqrt_apx(dx2[q] + hsqf);
                } else if (TAB == TAB2D) {
                    const float *row = tab + dy1 * N0;
#pragma unroll
                    for (int q = 0; q < NC; ++q) {
                        const int dx = (int)base_dx + q;
                        cst[q] = __ldg(row + (dx < 0 ? -dx : dx));
                    }
                } else {
                    const float *row = tab + hsq;
#pragma unroll
                    for (int q = 0; q < NC; ++q) {
                        const int dx = (int)base_dx + q;
                        cst[q] = __ldg(row + dx * dx);
                    }
                }
                const float *mrow = mus + th * M_X;
#pragma unroll
                for (int kk = 0; kk < KR; ++kk) {
#pragma unroll
                    for (int tx = 0; tx < KAPPA; ++tx) {
                        const float m = mrow[kk * KAPPA + tx];
#pragma unroll
                        for (int r = 0; r < CF_R; ++r)
                            acc[kk][r] = fmaf(m, cst[kk * KAPPA + tx - r + CF_R - 1], acc[kk][r]);
                    }
                }
            }
            // fold columns into their blocks: numer[kk][l] += sum_r nu_c * G
            const int64_t cbase = cx0 + hrow * N0;
            float nv[CF_R];
#pragma unroll
            for (int r = 0; r < CF_R; ++r) nv[r] = (float)nub[cbase + r];
            int64_t l_hi = 0;
#pragma unroll
            for (int a = nd - 1; a >= 1; --a) l_hi = l_hi * c.n[a] + chc[a] / KAPPA;
#pragma unroll
            for (int kk = 0; kk < KR; ++kk) {
                if (kk >= kr_valid) break;
                constexpr int PER = KAPPA < CF_R ? KAPPA : CF_R;  // columns per block in segment
#pragma unroll
                for (int g = 0; g < CF_R / PER; ++g) {
                    float s = 0.f;
#pragma unroll
                    for (int r = g * PER; r < (g + 1) * PER; ++r) s = fmaf(nv[r], acc[kk][r], s);
                    const int64_t lx = (cx0 + g * PER) / KAPPA;
                    atomicAdd(&numer[kk * n + l_hi * n0 + lx], (double)s);
                }
            }
        }
    }
    __syncthreads();
    // C-bar = numer / (mu~ nu~) or the centre cost where that product is 0
    for (int64_t i = threadIdx.x; i < (int64_t)kr_valid * n; i += CF_THREADS) {
        const int kk = (int)(i / n);
        const int64_t l = i - kk * n;
        const int64_t k = k_hi * n0 + kx0 + kk;
        const double denom = __dmul_rn(mu_c[b * n + k], nu_c[b * n + l]);
        const int64_t oi = (b * n + k) * n + l;
        const bool un = denom == 0.0;
        out[oi] = un ? Ccentre[k * n + l] : numer[i] / denom;
        if (unused) unused[oi] = un ? 1 : 0;
    }
}

template <int KAPPA, int KR>
static int launch_kappa(const double *mu, const double *nu, const double *mu_c, const double *nu_c,
                        const double *Ccentre, const double *table, int64_t max_sq, double *out,
                        uint8_t *unused, int64_t batch, const Grid &f, const Grid &c, bool p1,
                        cudaStream_t st) {
    const int64_t n = c.cells;
    int m_hi = 1;
    for (int a = 1; a < f.nd; ++a) m_hi *= KAPPA;
    const size_t bytes = sizeof(double) * KR * n + sizeof(float) * m_hi * KAPPA * KR;
    if (bytes > 200 * 1024) return GDT_ERR_UNSUPPORTED;
    const bool two_d = f.nd == 2;
    const int64_t tcount = p1 ? 1 : (two_d ? f.n[0] * f.n[1] : max_sq + 1);
    float *ftab = nullptr;
    if (malloc_async(reinterpret_cast<void **>(&ftab), sizeof(float) * tcount, st) != cudaSuccess) return GDT_ERR_CUDA;
    if (p1) {
    } else if (two_d)
        ftable2d_kernel<<<grid_size(tcount, 256), 256, 0, st>>>(table, ftab, f.n[1], f.n[0]);
    else
        ftable1d_kernel<<<grid_size(tcount, 256), 256, 0, st>>>(table, ftab, tcount);
    const int64_t tiles_x = (c.n[0] + KR - 1) / KR;
    dim3 grid((unsigned)(tiles_x * (n / c.n[0])), (unsigned)batch);
    auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        kern<<<grid, CF_THREADS, bytes, st>>>(mu, nu, mu_c, nu_c, Ccentre, ftab, out, unused, f, c);
    };
    if (p1) {
        if (f.nd == 1) run(cbar_toeplitz_kernel<KAPPA, KR, 1, true>);
        else if (f.nd == 2) run(cbar_toeplitz_kernel<KAPPA, KR, 2, true>);
        else if (f.nd == 3) run(cbar_toeplitz_kernel<KAPPA, KR, 3, true>);
    } else {
        if (f.nd == 1) run(cbar_toeplitz_kernel<KAPPA, KR, 1, false>);
        else if (f.nd == 2) run(cbar_toeplitz_kernel<KAPPA, KR, 2, false>);
        else if (f.nd == 3) run(cbar_toeplitz_kernel<KAPPA, KR, 3, false>);
    }
    cudaFreeAsync(ftab, st);
    return GDT_OK;
}

// Returns GDT_ERR_UNSUPPORTED when the shape is outside the tiled kernel's
// envelope (caller falls back to the generic tile kernel).
int cbar_fast_toeplitz(const double *mu, const double *nu, const double *mu_c,
                       const double *nu_c, const double *Ccentre, const double *table,
                       int64_t max_sq, double *out, uint8_t *unused, int64_t batch, const Grid &f,
                       const Grid &c, int kappa, double p, cudaStream_t st) {
    const bool p1 = p == 1.0;
    if (table == nullptr || f.n[0] % CF_R != 0 || f.n[0] / CF_R > CF_THREADS)
        return GDT_ERR_UNSUPPORTED;
    if (ipow(kappa, f.nd) > 64 || f.nd > 3) return GDT_ERR_UNSUPPORTED;  // fp32 bound: 64 ulp
    switch (kappa) {
        case 2: return launch_kappa<2, 8>(mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused,
                                          batch, f, c, p1, st);
        case 4: return launch_kappa<4, 4>(mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused,
                                          batch, f, c, p1, st);
        case 8: return launch_kappa<8, 2>(mu, nu, mu_c, nu_c, Ccentre, table, max_sq, out, unused,
                                          batch, f, c, p1, st);
        default: return GDT_ERR_UNSUPPORTED;
    }
}

}  // namespace gdt
