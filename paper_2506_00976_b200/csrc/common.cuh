// Shared helpers for the gridot_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gridot_b200.h"

namespace gdt {

// Error text of the last failing call on this host thread (gdt_last_error).
void set_error(const std::string &msg);
int cuda_status(const char *where);  // GDT_OK or GDT_ERR_CUDA after a launch
cudaError_t malloc_async(void **p, size_t bytes, cudaStream_t st);  // pooled workspace

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Fine grid with axis-0-fastest flat order (measures.py:3-6).
struct Grid {
    int nd;
    int64_t n[GDT_MAX_DIM];
    int64_t stride[GDT_MAX_DIM];
    int64_t cells;
};

inline bool make_grid(Grid &g, int ndim, const int64_t *dims) {
    if (ndim < 1 || ndim > GDT_MAX_DIM || dims == nullptr) return false;
    g.nd = ndim;
    int64_t s = 1;
    for (int a = 0; a < GDT_MAX_DIM; ++a) {
        if (a < ndim) {
            if (dims[a] < 1) return false;
            g.n[a] = dims[a];
            g.stride[a] = s;
            s *= dims[a];
        } else {
            g.n[a] = 1;
            g.stride[a] = s;
        }
    }
    g.cells = s;
    return true;
}

// Coarse grid of a kappa-divisible fine grid.
inline bool make_coarse(Grid &c, const Grid &f, int kappa) {
    int64_t d[GDT_MAX_DIM];
    for (int a = 0; a < f.nd; ++a) {
        if (kappa < 1 || f.n[a] % kappa) return false;
        d[a] = f.n[a] / kappa;
    }
    return make_grid(c, f.nd, d);
}

__host__ __device__ inline int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e-- > 0) r *= b;
    return r;
}

inline unsigned grid_size(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 0x7fffffff) g = 0x7fffffff;
    return (unsigned)g;
}

// rho^p from an integer squared distance, matching numpy's `sq ** (p/2)`
// fast paths (p == 2 -> sq, p == 1 -> IEEE sqrt) and, for other p, the
// host-computed table of the same expression (costs.py:44-53).
__device__ __forceinline__ double cost_from_sq(int64_t sq, double p, const double *table) {
    if (p == 2.0) return (double)sq;
    if (p == 1.0) return __dsqrt_rn((double)sq);
    return table[sq];
}

// Numpy's float64 pairwise summation over n values v[0..n-1] read through
// `at(i)` (numpy/_core/src/umath/loops_utils.h.src, DOUBLE_pairwise_sum).
// Non-recursive form for n <= 128, recursive split above.
template <typename F>
__device__ double np_pairwise_small(F at, int64_t lo, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, at(lo + i));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = at(lo + j);
    int64_t i = 8;
    const int64_t stop = n - (n % 8);
    for (; i < stop; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], at(lo + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, at(lo + i));
    return res;
}

template <typename F>
__device__ double np_pairwise_rec(F at, int64_t lo, int64_t n) {
    if (n <= 128) return np_pairwise_small(at, lo, n);
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise_rec(at, lo, n2), np_pairwise_rec(at, lo + n2, n - n2));
}

template <typename F>
__device__ __forceinline__ double np_pairwise(F at, int64_t n) {
    return n <= 128 ? np_pairwise_small(at, 0, n) : np_pairwise_rec(at, 0, n);
}

// fp64 block reduction helper (any order; used where BLAS ddot / numpy
// sums have no fixed order the reference depends on).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int THREADS>
__device__ double block_sum(double v, double *sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = lane < THREADS / 32 ? sh[lane] : 0.0;
        r = warp_sum(r);
        if (lane == 0) sh[0] = r;
    }
    __syncthreads();
    r = sh[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}

__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// One source row of a lane's 8 x 8 candidate block from the 16 table floats
// L: the cost of offset index q is L[q] (off >= 0) or L[14 - q] (off < 0).
// Each add.f32x2 pairs the candidates of ONE source s for two adjacent
// outputs r8, r8 + 1: their costs cst[q] and cst[q - 1] (q = s - r8 + 7) are
// an aligned register pair of L (straight or swapped) and the potential vs[s]
// is the broadcast scalar operand -- no register shuffling.  Per source the
// aligned output pairs are (0,1),(2,3),(4,5),(6,7) or (1,2),(3,4),(5,6) plus
// two scalar adds, depending on the parity of s (and on the direction).
template <bool REV, bool SUB>
__device__ __forceinline__ void minplus_row8(const float (&L)[16], const float (&vs)[8],
                                             float (&best)[8]) {
    float cand[8][8];  // [r8][s], consumed by the min folds below
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        // pairs (r8, r8+1) whose cost pair is aligned: straight L pair
        // (L[q-1], L[q]) needs q - 1 even; swapped pair (L[14-q], L[15-q])
        // needs 14 - q even
        const int first = REV ? ((s % 2 == 0) ? 1 : 0) : ((s % 2 == 0) ? 0 : 1);
#pragma unroll
        for (int r8 = first; r8 + 1 < 8; r8 += 2) {
            const int q = s - r8 + 7;
            unsigned long long c;
            if (!REV) c = pk2(L[q], L[q - 1]);        // (cst[q], cst[q-1])
            else c = pk2(L[14 - q], L[15 - q]);       // (cst[q], cst[q-1])
            unsigned long long rr;
            const unsigned long long vv = pk2(vs[s], vs[s]);
            if (SUB) asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(c), "l"(vv));
            else asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(c), "l"(vv));
            cand[r8][s] = __uint_as_float((unsigned)(rr & 0xffffffffu));
            cand[r8 + 1][s] = __uint_as_float((unsigned)(rr >> 32));
        }
        if (first == 1) {  // r8 = 0 and r8 = 7 left over for this s
            const float c0 = REV ? L[7 - s] : L[s + 7], c7 = REV ? L[14 - s] : L[s];
            cand[0][s] = SUB ? c0 - vs[s] : c0 + vs[s];
            cand[7][s] = SUB ? c7 - vs[s] : c7 + vs[s];
        }
    }
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8)
#pragma unroll
        for (int s = 0; s < 8; s += 2) best[r8] = fmin3(best[r8], cand[r8][s], cand[r8][s + 1]);
}

}  // namespace gdt

#define GDT_CHECK_ARG(cond, msg)              \
    do {                                      \
        if (!(cond)) {                        \
            gdt::set_error(msg);              \
            return GDT_ERR_ARG;               \
        }                                     \
    } while (0)
