// K9, p != 2: exact brute-force c-transform with conservative tile pruning.
//
//   out_j = min_i rho(x_i, x_j)^p - v_i          (quantized.py:450-484)
//
// Each warp owns a 16 x 16 (2-D) or 16 x 4 x 4 (3-D) region of outputs, a
// lane 8 consecutive outputs along axis 0.  Sources are cut into tiles of
// 8 x 8 (2-D) / 8 x 4 x 4 (3-D) cells with a precomputed max_i v_i per tile.
// A tile I can only improve an output j of the region J if
//     lb(I, J) = rho(gap(I, J))^p - max_{i in I} v_i  <  max_{j in J} best_j,
// where gap is the smallest grid distance between the two boxes; because
// rounding is monotone, lb is <= every rounded candidate C_ij - v_i of the
// tile, so skipping such tiles never changes the minimum.  The warp visits
// tiles in Chebyshev rings around its own region (near tiles first, which
// tightens max best_j quickly) and stops at the first ring whose smallest
// possible lb reaches the bound.  The result equals the full brute force
// bit for bit; the work shrinks with the regularity of v (potentials of
// transport problems are Lipschitz, so far tiles are pruned).
//
// Inner loop (fp32): for one source row of 8 cells a lane needs 15 distinct
// costs (Toeplitz: cost depends on dx only) and does 64 candidates with
// packed sub.f32x2 (FADD2) and 3-input min (FMNMX3).  p == 1 costs use
// sqrt.approx (fp32 mode contract: bounds within 1e-5); the pruning bound is
// lowered by 2^-20 to stay below every approximated cost.  fp64 reads the
// exact cost table (p = 1: IEEE sqrt of the integer squared distance).
#include "common.cuh"

namespace gdt {

__device__ __forceinline__ void sub_f32x2(float c0, float c1, float v0, float v1, float &r0,
                                          float &r1) {
    unsigned long long rr;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(pk2(c0, c1)), "l"(pk2(v0, v1)));
    r0 = __uint_as_float((unsigned)(rr & 0xffffffffu));
    r1 = __uint_as_float((unsigned)(rr >> 32));
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <typename T>
__global__ void tile_max_kernel(const T *__restrict__ v, T *__restrict__ tmax, int64_t batch,
                                Grid g, int s0, int s1, int s2) {
    const int64_t nt0 = g.n[0] / s0, nt1 = g.n[1] / s1, nt2 = g.n[2] / s2;
    const int64_t per = nt0 * nt1 * nt2;
    const int64_t total = batch * per;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / per;
        int64_t r = idx - b * per;
        const int64_t t0 = r % nt0;
        r /= nt0;
        const int64_t t1 = r % nt1, t2 = r / nt1;
        T m = (T)-INFINITY;
        for (int z = 0; z < s2; ++z)
            for (int y = 0; y < s1; ++y) {
                const T *row = v + b * g.cells + (t2 * s2 + z) * g.stride[2] +
                               (t1 * s1 + y) * g.stride[1] + t0 * s0;
                for (int x = 0; x < s0; ++x) m = row[x] > m ? row[x] : m;
            }
        tmax[idx] = m;
    }
}

// ND = 2: region 16x16, tile 8x8; ND = 3: region 16x4x4, tile 8x4x4
template <typename T, int ND, bool P1>
__global__ void __launch_bounds__(64) pruned_ct_kernel(const T *__restrict__ v,
                                                        const T *__restrict__ tmax,
                                                        T *__restrict__ out, int64_t batch,
                                                        Grid g, const T *__restrict__ tab,
                                                        unsigned long long *__restrict__ counter,
                                                        const T *__restrict__ tab2, int W2) {
    constexpr int R1 = ND == 2 ? 16 : 4, R2 = ND == 2 ? 1 : 4;   // region extent y, z
    constexpr int S1 = ND == 2 ? 8 : 4, S2 = ND == 2 ? 1 : 4;    // tile extent y, z
    const int lane = threadIdx.x & 31;
    const int nr0 = (int)(g.n[0] / 16), nr1 = (int)(g.n[1] / R1), nr2 = (int)(g.n[2] / R2);
    const int64_t regions = (int64_t)nr0 * nr1 * nr2;
    const int64_t total = batch * regions;
    // one region per 2-warp CTA; warp `half` takes every other tile of each
    // ring (with its own bound), the two results are merged at the end.  Many
    // small CTAs let the hardware scheduler balance the uneven pruned work.
    (void)counter;
    const int half = threadIdx.x >> 5;
    const int64_t warp = blockIdx.x;
    if (warp >= total) return;
    __shared__ T other[32][8];
    int parity = 0;
    const int64_t b = warp / regions;
    int rr = (int)(warp - b * regions);
    const int rx = rr % nr0;
    rr /= nr0;
    const int ry = rr % nr1, rz = rr / nr1;
    const int X0 = rx * 16, Y0 = ry * R1, Z0 = rz * R2;
    const int xj0 = X0 + 8 * (lane & 1);
    const int yj = Y0 + ((lane >> 1) % R1);
    const int zj = Z0 + (ND == 3 ? (lane >> 3) : 0);
    const T *vb = v + b * g.cells;
    const int nt0 = (int)(g.n[0] / 8), nt1 = (int)(g.n[1] / S1), nt2 = (int)(g.n[2] / S2);
    const T *tm = tmax + b * (int64_t)nt0 * nt1 * nt2;

    // max of v over the pair (termination bound)
    T vall = (T)-INFINITY;
    for (int i = lane; i < nt0 * nt1 * nt2; i += 32) vall = tm[i] > vall ? tm[i] : vall;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T w = __shfl_xor_sync(0xffffffffu, vall, o);
        vall = w > vall ? w : vall;
    }

    T best[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) best[r] = (T)INFINITY;
    T ub = (T)INFINITY;

    // home box in tile units
    const int h0lo = X0 / 8, h0hi = (X0 + 15) / 8;
    const int h1lo = Y0 / S1, h1hi = (Y0 + R1 - 1) / S1;
    const int h2lo = Z0 / S2, h2hi = (Z0 + R2 - 1) / S2;
    const int rmax = max(max(nt0, nt1), nt2);
    constexpr int smin = ND == 2 ? 8 : 4;

    auto lowered = [](T c) -> T {
        if constexpr (P1 && sizeof(T) == 4) return c * (1.0f - 1.0f / 1048576.0f);
        else return c;
    };
    auto cost_of = [&](int sq) -> T {
        if constexpr (sizeof(T) == 4) {
            if constexpr (P1) return sqrt_approx((float)sq);
            else return __ldg(tab + sq);
        } else {
            return __ldg(tab + sq);
        }
    };

    for (int r = 0; r <= rmax; ++r) {
        if (r >= 1) {  // smallest lb any tile of ring r can have
            const int gap = (r - 1) * smin + 1;
            const T lb = lowered(cost_of(gap * gap)) - vall;
            if (lb >= ub) break;
        }
        const int a0 = max(h0lo - r, 0), b0 = min(h0hi + r, nt0 - 1);
        const int a1 = max(h1lo - r, 0), b1 = min(h1hi + r, nt1 - 1);
        const int a2 = max(h2lo - r, 0), b2 = min(h2hi + r, nt2 - 1);
        for (int t2 = a2; t2 <= b2; ++t2)
            for (int t1 = a1; t1 <= b1; ++t1) {
                const int d1 = t1 < h1lo ? h1lo - t1 : (t1 > h1hi ? t1 - h1hi : 0);
                const int d2 = t2 < h2lo ? h2lo - t2 : (t2 > h2hi ? t2 - h2hi : 0);
                // only ring tiles: a full t0 sweep on the ring's t1/t2 faces, else
                // just the two t0 ends at distance r
                const bool face = max(d1, d2) == r;
                const int step = face ? 1 : (h0hi + r) - (h0lo - r);
                for (int t0 = face ? a0 : h0lo - r; t0 <= b0; t0 += step > 0 ? step : 1) {
                    if (t0 < a0) continue;
                    const int d0 = t0 < h0lo ? h0lo - t0 : (t0 > h0hi ? t0 - h0hi : 0);
                    if (max(max(d0, d1), d2) != r) continue;
                    // gap between the region box and the tile box, per axis
                    const int g0 = max(0, max(t0 * 8 - (X0 + 15), X0 - (t0 * 8 + 7)));
                    const int g1 = max(0, max(t1 * S1 - (Y0 + R1 - 1), Y0 - (t1 * S1 + S1 - 1)));
                    const int g2 = max(0, max(t2 * S2 - (Z0 + R2 - 1), Z0 - (t2 * S2 + S2 - 1)));
                    const T lb = lowered(cost_of(g0 * g0 + g1 * g1 + g2 * g2)) -
                                 tm[((int64_t)t2 * nt1 + t1) * nt0 + t0];
                    if (((parity++) & 1) != half) continue;
                    if (lb >= ub) continue;
                    const int sx0 = t0 * 8;
                    // dx^2 of the 15 Toeplitz slots, fixed for the whole tile
                    float dx2[15];
#pragma unroll
                    for (int q = 0; q < 15; ++q) {
                        const float dx = (float)(sx0 - xj0 - 7 + q);
                        dx2[q] = dx * dx;
                    }
                    for (int z = 0; z < S2; ++z)
                        for (int y = 0; y < S1; ++y) {
                            const int ys = t1 * S1 + y, zs = t2 * S2 + z;
                            const int hsq = (ys - yj) * (ys - yj) + (zs - zj) * (zs - zj);
                            const T *row = vb + (int64_t)zs * g.stride[2] + (int64_t)ys * g.stride[1] + sx0;
                            T vs[8];
                            if constexpr (sizeof(T) == 4) {
                                const float4 v0 = __ldg(reinterpret_cast<const float4 *>(row));
                                const float4 v1 = __ldg(reinterpret_cast<const float4 *>(row) + 1);
                                vs[0] = v0.x; vs[1] = v0.y; vs[2] = v0.z; vs[3] = v0.w;
                                vs[4] = v1.x; vs[5] = v1.y; vs[6] = v1.z; vs[7] = v1.w;
                            } else {
#pragma unroll
                                for (int s = 0; s < 8; ++s) vs[s] = row[s];
                            }
                            T cst[15];
                            if constexpr (sizeof(T) == 4 && P1) {
                                const float hf = (float)hsq;
#pragma unroll
                                for (int q = 0; q < 15; ++q) cst[q] = sqrt_approx(dx2[q] + hf);
                            } else if (ND == 2 && tab2 != nullptr) {
                                // 2-D table row |dy|: the 15 costs of a lane are
                                // consecutive |dx| entries (coalesced per lane)
                                const int dyy = ys > yj ? ys - yj : yj - ys;
                                const T *trow = tab2 + (int64_t)dyy * W2;
#pragma unroll
                                for (int q = 0; q < 15; ++q) {
                                    const int dx = sx0 - xj0 - 7 + q;
                                    cst[q] = __ldg(trow + (dx < 0 ? -dx : dx));
                                }
                            } else {
#pragma unroll
                                for (int q = 0; q < 15; ++q) {
                                    const int dx = sx0 - xj0 - 7 + q;
                                    cst[q] = cost_of(hsq + dx * dx);
                                }
                            }
                            if constexpr (sizeof(T) == 4) {
#pragma unroll
                                for (int r8 = 0; r8 < 8; ++r8) {
#pragma unroll
                                    for (int s = 0; s < 8; s += 2) {
                                        float c0, c1;
                                        sub_f32x2(cst[s - r8 + 7], cst[s + 1 - r8 + 7], vs[s],
                                                  vs[s + 1], c0, c1);
                                        best[r8] = fmin3(best[r8], c0, c1);
                                    }
                                }
                            } else {
#pragma unroll
                                for (int r8 = 0; r8 < 8; ++r8)
#pragma unroll
                                    for (int s = 0; s < 8; ++s)
                                        best[r8] = fmin(best[r8], __dsub_rn(cst[s - r8 + 7], vs[s]));
                            }
                        }
                    // refresh the warp bound max_j best_j
                    T m = best[0];
#pragma unroll
                    for (int r8 = 1; r8 < 8; ++r8) m = best[r8] > m ? best[r8] : m;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const T w = __shfl_xor_sync(0xffffffffu, m, o);
                        m = w > m ? w : m;
                    }
                    ub = m;
                }
            }
    }
    if (half == 1) {
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) other[lane][r8] = best[r8];
    }
    __syncthreads();
    if (half == 0) {
        T *ob = out + b * g.cells + (int64_t)zj * g.stride[2] + (int64_t)yj * g.stride[1] + xj0;
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
            const T o = other[lane][r8];
            ob[r8] = o < best[r8] ? o : best[r8];
        }
    }
}

// ---- fp32, p = 1, 2-D grids up to 128 x 128: shared-memory cost table -----
//
// Same regions, tiles, ring order and pruning rule as pruned_ct_kernel, but the
// 15 Toeplitz costs of a (lane, source row) pair come from a per-CTA table of
// correctly rounded sqrt(dx^2 + dy^2) instead of 15 MUFU sqrt.approx (the MUFU
// pipe bounded the kernel).  Row |dy| of the table holds T[i] = cost(|i - 7|, dy)
// for i in [0, 135]: for a lane whose 8 outputs start at xj0 and a tile row
// starting at sx0, off = sx0 - xj0 is a multiple of 8 and the lane's costs are
// T[off + q] (off >= 0) or T[-off + 14 - q] (off < 0), q = 0..14 -- 16 aligned
// floats, four LDS.128.  Row stride 140 floats (12 mod 32 banks) makes the
// 16-byte reads of 8 lanes on 8 different rows conflict-free.
//
// Work distribution (round 2): a region is shared by CT_TAB_WPR warps that
// take its ring-ordered tiles from one cursor, and their per-output minima
// live in one shared array (atomicMin on order-preserving integer keys), so
// every warp prunes against the region's best known bound, not only its own.
// Many warps per region finish a region fast; with ~1.2 regions per warp pair
// (the round-1 mapping) the SMs idled behind the slowest regions (ncu: SM
// active ~42%).  Regions come from a global counter (persistent CTAs).  The
// result equals the brute force bit for bit: a tile is skipped only when its
// lower bound reaches the largest current best of the region.
constexpr int CT_TAB_W = 140;      // row stride (floats)
constexpr int CT_TAB_ROWS = 128;   // |dy| <= 127
constexpr int CT_TAB_WPR = 4;      // warps per region
constexpr int CT_TAB_REG = 4;      // regions per CTA
constexpr int CT_TAB_CH = 8;       // tiles a warp takes from the region's cursor at a time
constexpr int CT_TAB_GT = 32 * CT_TAB_WPR;  // threads of a region group

__device__ __forceinline__ void group_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(CT_TAB_GT) : "memory");
}

// float <-> int key with the same order (for atomicMin on shared memory)
__device__ __forceinline__ int ord_key(float x) {
    const int i = __float_as_int(x);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord_val(int k) {
    return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff);
}

constexpr int CT_TAB_TILES = 256;  // (128 / 8)^2 source tiles at most

#ifdef GDT_IPF_TRACE
// debug builds: source tiles evaluated exactly / visited by the table kernel
__device__ unsigned long long g_ct_tiles[2];
#endif

__global__ void __launch_bounds__(CT_TAB_GT * CT_TAB_REG, 2) pruned_ct_tab_kernel(
    const float *__restrict__ v, const float *__restrict__ tmax, float *__restrict__ out,
    int64_t batch, Grid g, unsigned long long *__restrict__ counter) {
    extern __shared__ __align__(16) float ct_tab[];  // [CT_TAB_ROWS][CT_TAB_W]
    __shared__ int sbest[CT_TAB_REG][256];           // region minima (ord_key)
    __shared__ long long next_region[CT_TAB_REG];
    // per region group: the region's tiles in Chebyshev-ring order, packed
    // (ring << 16) | tile, and the cursor its warps take tiles from
    __shared__ unsigned tiles_s[CT_TAB_REG][CT_TAB_TILES];
    __shared__ int ring_cnt[CT_TAB_REG][17];
    __shared__ int cursor[CT_TAB_REG];
    const int lane = threadIdx.x & 31;
    const int warp_in_cta = threadIdx.x >> 5;
    const int slot = warp_in_cta / CT_TAB_WPR;
    const int pt = threadIdx.x % CT_TAB_GT;  // thread index inside the group
    const int bar_id = 1 + slot;             // named barrier of this group
    const int N0 = (int)g.n[0], N1 = (int)g.n[1];
    // table: row dy, column i -> sqrt((i - 7)^2 + dy^2), correctly rounded
    for (int e = threadIdx.x; e < CT_TAB_ROWS * CT_TAB_W; e += blockDim.x) {
        const int dy = e / CT_TAB_W, i = e - dy * CT_TAB_W;
        const int dx = i - 7;
        ct_tab[e] = sqrtf((float)(dx * dx + dy * dy));
    }
    __syncthreads();

    const int nr0 = N0 / 16, nr1 = N1 / 16;
    const int64_t regions = (int64_t)nr0 * nr1;
    const int64_t total = batch * regions;
    const int nt0 = N0 / 8, nt1 = N1 / 8, ntiles = nt0 * nt1;
    constexpr int PER = (CT_TAB_TILES + CT_TAB_GT - 1) / CT_TAB_GT;  // tiles per thread (sort)
    for (;;) {
        if (pt == 0) next_region[slot] = (long long)atomicAdd(counter, 1ull);
        if (pt < 17) ring_cnt[slot][pt] = 0;
        for (int i = pt; i < 256; i += CT_TAB_GT) sbest[slot][i] = ord_key(INFINITY);
        group_sync(bar_id);
        const int64_t region = next_region[slot];
        if (region >= total) break;
        const int64_t b = region / regions;
        const int rr = (int)(region - b * regions);
        const int rx = rr % nr0, ry = rr / nr0;
        const int X0 = rx * 16, Y0 = ry * 16;
        const int h0lo = X0 / 8, h0hi = h0lo + 1, h1lo = Y0 / 8, h1hi = h1lo + 1;
        // ring of every tile, counting sort into ring order
        int my_ring[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int t = pt + CT_TAB_GT * q;
            my_ring[q] = -1;
            if (t < ntiles) {
                const int t0 = t % nt0, t1 = t / nt0;
                const int d0 = t0 < h0lo ? h0lo - t0 : (t0 > h0hi ? t0 - h0hi : 0);
                const int d1 = t1 < h1lo ? h1lo - t1 : (t1 > h1hi ? t1 - h1hi : 0);
                my_ring[q] = max(d0, d1);
                atomicAdd(&ring_cnt[slot][my_ring[q]], 1);
            }
        }
        group_sync(bar_id);
        if (pt == 0) {
            int acc = 0;
            for (int r = 0; r < 17; ++r) {
                const int c = ring_cnt[slot][r];
                ring_cnt[slot][r] = acc;
                acc += c;
            }
            cursor[slot] = 0;
        }
        group_sync(bar_id);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int t = pt + CT_TAB_GT * q;
            if (my_ring[q] >= 0) {
                const int pos = atomicAdd(&ring_cnt[slot][my_ring[q]], 1);
                tiles_s[slot][pos] = ((unsigned)my_ring[q] << 16) |
                                     ((unsigned)(t / nt0) << 8) | (unsigned)(t % nt0);
            }
        }
        group_sync(bar_id);

        float best[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) best[r] = INFINITY;
        // lanes 0-15: rows Y0.., left 8 columns; lanes 16-31: right 8 columns
        // (the 8 lanes of a quarter warp read 8 different table rows: with a
        // row stride of 12 mod 32 banks their 16-byte reads do not conflict)
        const int xj0 = X0 + 8 * (lane >> 4);
        const int yj = Y0 + (lane & 15);
        int *sb = sbest[slot] + (lane & 15) * 16 + 8 * (lane >> 4);  // this lane's 8 outputs
        const float *vb = v + b * g.cells;
        const float *tm = tmax + b * (int64_t)ntiles;
        float vall = -INFINITY;
        for (int i = lane; i < ntiles; i += 32) vall = fmaxf(vall, tm[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vall = fmaxf(vall, __shfl_xor_sync(0xffffffffu, vall, o));
        float ub = INFINITY;
        // Tiles are taken CT_TAB_CH at a time: lane l of the warp examines tile
        // idx + l (its pruning bound and its ring's bound, all in one pass),
        // then the warp walks the chunk in ring order with the bound it keeps
        // tightening.  One cursor atomic and one round of table / tile-max loads
        // per chunk instead of per tile.
        bool done = false;
        while (!done) {
            int idx = 0;
            if (lane == 0) idx = atomicAdd(&cursor[slot], CT_TAB_CH);
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx >= ntiles) break;
            unsigned e_l = 0xffffffffu;
            float lb_l = INFINITY, rb_l = -INFINITY;
            if (lane < CT_TAB_CH && idx + lane < ntiles) {
                e_l = tiles_s[slot][idx + lane];
                const int r = (int)(e_l >> 16), t1 = (int)((e_l >> 8) & 0xffu), t0 = (int)(e_l & 0xffu);
                if (r >= 1) {  // smallest cost any tile of ring r can have, minus max v
                    const int gap = (r - 1) * 8 + 1;
                    rb_l = (gap + 7 < CT_TAB_W ? ct_tab[gap + 7] : sqrtf((float)gap * gap)) - vall;
                }
                const int g0 = max(0, max(t0 * 8 - (X0 + 15), X0 - (t0 * 8 + 7)));
                const int g1 = max(0, max(t1 * 8 - (Y0 + 15), Y0 - (t1 * 8 + 7)));
                lb_l = ct_tab[g1 * CT_TAB_W + g0 + 7] - tm[t1 * nt0 + t0];
            }
#pragma unroll 1
            for (int k = 0; k < CT_TAB_CH; ++k) {
                const unsigned e = __shfl_sync(0xffffffffu, e_l, k);
                if (e == 0xffffffffu) break;  // past the last tile
                const float rb = __shfl_sync(0xffffffffu, rb_l, k);
                if (rb >= ub) {  // no tile of this ring or a later one can improve the region
                    done = true;
                    break;
                }
                const float lb = __shfl_sync(0xffffffffu, lb_l, k);
                const int t1 = (int)((e >> 8) & 0xffu), t0 = (int)(e & 0xffu);
#ifdef GDT_IPF_TRACE
                if (lane == 0) atomicAdd(&g_ct_tiles[1], 1ull);
                if (lane == 0 && !(lb >= ub)) atomicAdd(&g_ct_tiles[0], 1ull);
#endif
                if (lb >= ub) continue;
            const int sx0 = t0 * 8, off = sx0 - xj0;
            const int base = off >= 0 ? off : -off;
            const float *vrow = vb + (int64_t)(t1 * 8) * N0 + sx0;
            // the next row's potentials are loaded before this row's min-plus
            float4 v0 = __ldg(reinterpret_cast<const float4 *>(vrow));
            float4 v1 = __ldg(reinterpret_cast<const float4 *>(vrow) + 1);
            // (two rows per trip: the prefetched potentials alternate between two
            // register sets instead of being copied every row -- 8 moves of 94
            // instructions per row)
#pragma unroll 2
            for (int y = 0; y < 8; ++y) {
                const int ys = t1 * 8 + y;
                const int dy = ys > yj ? ys - yj : yj - ys;
                const float4 *trow = reinterpret_cast<const float4 *>(ct_tab + dy * CT_TAB_W + base);
                float L[16];
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    const float4 tt = trow[c4];
                    L[4 * c4] = tt.x;
                    L[4 * c4 + 1] = tt.y;
                    L[4 * c4 + 2] = tt.z;
                    L[4 * c4 + 3] = tt.w;
                }
                const float vs[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                if (y + 1 < 8) {
                    v0 = __ldg(reinterpret_cast<const float4 *>(vrow + (y + 1) * N0));
                    v1 = __ldg(reinterpret_cast<const float4 *>(vrow + (y + 1) * N0) + 1);
                }
                if (off >= 0) minplus_row8<false, true>(L, vs, best);
                else minplus_row8<true, true>(L, vs, best);
            }
            // publish to the region's minima, take the others' back, and
            // refresh this warp's bound: the largest best of the region
            float m = -INFINITY;
#pragma unroll
            for (int r8 = 0; r8 < 8; ++r8) {
                const int got = atomicMin(sb + r8, ord_key(best[r8]));
                best[r8] = fminf(best[r8], ord_val(got));
                m = fmaxf(m, best[r8]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            ub = m;
            }
        }
        group_sync(bar_id);  // every warp's minima are in sbest
        if (warp_in_cta % CT_TAB_WPR == 0) {
            float *ob = out + b * g.cells + (int64_t)yj * N0 + xj0;
#pragma unroll
            for (int r8 = 0; r8 < 8; ++r8) ob[r8] = ord_val(sb[r8]);
        }
        group_sync(bar_id);  // the group's shared lists are reused by the next region
    }
}

// T2[|dy|][|dx|] = tab[dx^2 + dy^2] (the same values, laid out by axis offsets)
template <typename T>
__global__ void ct_cost2d_kernel(const T *__restrict__ tab, int W, T *__restrict__ t2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W * W; i += gridDim.x * blockDim.x) {
        const int a = i / W, bx = i - a * W;
        t2[i] = tab[(int64_t)a * a + (int64_t)bx * bx];
    }
}

// Returns GDT_ERR_UNSUPPORTED outside the tiled envelope (caller falls back).
// v: device input of type T (fp32 path expects an fp32 copy); tab: T cost table
// by squared distance (unused for fp32 p == 1); tmax: scratch [batch * tiles].
template <typename T>
static int run_pruned(const T *v, T *out, T *tmax, int64_t batch, const Grid &g, double p,
                      const T *tab, cudaStream_t st) {
    const bool p1 = p == 1.0;
    int s1, s2;
    if (g.nd == 2) {
        if (g.n[0] % 16 || g.n[1] % 16) return GDT_ERR_UNSUPPORTED;
        s1 = 8;
        s2 = 1;
    } else if (g.nd == 3) {
        if (g.n[0] % 16 || g.n[1] % 4 || g.n[2] % 4) return GDT_ERR_UNSUPPORTED;
        s1 = 4;
        s2 = 4;
    } else {
        return GDT_ERR_UNSUPPORTED;
    }
    const int64_t tiles = (g.n[0] / 8) * (g.n[1] / s1) * (g.n[2] / s2);
    tile_max_kernel<T><<<grid_size(batch * tiles, 128), 128, 0, st>>>(v, tmax, batch, g, 8, s1, s2);
    const int64_t regions = (g.n[0] / 16) * (g.n[1] / (g.nd == 2 ? 16 : 4)) *
                            (g.n[2] / (g.nd == 2 ? 1 : 4));
    const int64_t warps = batch * regions;
    unsigned long long *counter =
        reinterpret_cast<unsigned long long *>(tmax + ((batch * tiles + 1) & ~1ll));
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    (void)sms;
    const unsigned ctas = (unsigned)warps;  // one region per 2-warp CTA
    if constexpr (sizeof(T) == 4) {
        if (g.nd == 2 && p1 && g.n[0] <= CT_TAB_ROWS && g.n[1] <= CT_TAB_ROWS) {
            const size_t tb = sizeof(float) * CT_TAB_ROWS * CT_TAB_W;
            cudaFuncSetAttribute(pruned_ct_tab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tb);
            int dev2 = 0, nsm = 148;
            cudaGetDevice(&dev2);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev2);
            const int64_t need = (warps + CT_TAB_REG - 1) / CT_TAB_REG;
            const unsigned tctas = (unsigned)std::min<int64_t>(need, 2 * nsm);  // persistent
            pruned_ct_tab_kernel<<<tctas, CT_TAB_GT * CT_TAB_REG, tb, st>>>(
                reinterpret_cast<const float *>(v), reinterpret_cast<const float *>(tmax),
                reinterpret_cast<float *>(out), batch, g, counter);
            return GDT_OK;
        }
    }
    if (g.nd == 2) {
        // (a 2-D |dy| x |dx| table for the fp64 costs was measured slower than
        // the 1-D table by squared distance: 2.7 vs 1.75 ms per transform)
        T *t2 = nullptr;
        const int W2 = 0;
        if (p1 && sizeof(T) == 4)
            pruned_ct_kernel<T, 2, true><<<ctas, 64, 0, st>>>(v, tmax, out, batch, g, tab, counter,
                                                              nullptr, 0);
        else
            pruned_ct_kernel<T, 2, false><<<ctas, 64, 0, st>>>(v, tmax, out, batch, g, tab, counter,
                                                               t2, W2);
        if (t2) cudaFreeAsync(t2, st);
    } else {
        if (p1 && sizeof(T) == 4) pruned_ct_kernel<T, 3, true><<<ctas, 64, 0, st>>>(v, tmax, out, batch, g, tab, counter, nullptr, 0);
        else pruned_ct_kernel<T, 3, false><<<ctas, 64, 0, st>>>(v, tmax, out, batch, g, tab, counter, nullptr, 0);
    }
    return GDT_OK;
}

int ct_pruned_f32(const float *v, float *out, float *tmax, int64_t batch, const Grid &g, double p,
                  const float *ftab, cudaStream_t st) {
    return run_pruned<float>(v, out, tmax, batch, g, p, ftab, st);
}

int ct_pruned_f64(const double *v, double *out, double *tmax, int64_t batch, const Grid &g,
                  double p, const double *tab, cudaStream_t st) {
    return run_pruned<double>(v, out, tmax, batch, g, p, tab, st);
}

int64_t ct_pruned_tiles(const Grid &g) {
    if (g.nd == 2) return (g.n[0] / 8) * (g.n[1] / 8);
    if (g.nd == 3) return (g.n[0] / 8) * (g.n[1] / 4) * (g.n[2] / 4);
    return 0;
}

}  // namespace gdt

#ifdef GDT_IPF_TRACE
extern "C" int gdt_debug_ct_tiles(unsigned long long *host, int reset) {
    if (reset) {
        const unsigned long long z[2] = {0, 0};
        return cudaMemcpyToSymbol(gdt::g_ct_tiles, z, sizeof(z)) == cudaSuccess ? 0 : -1;
    }
    return cudaMemcpyFromSymbol(host, gdt::g_ct_tiles, sizeof(unsigned long long) * 2) ==
                   cudaSuccess
               ? 0
               : -1;
}
#endif
