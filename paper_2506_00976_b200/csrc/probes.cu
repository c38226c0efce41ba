// CUDA-core peak probes: the measured denominators of the FP32 / FP64
// rooflines bench.py reports (C-bar, c-transform, exact IPF).
//
// Each thread runs CHAINS independent dependent FMA chains, unrolled UNROLL
// times per loop trip, so the loop overhead is < 1% of the issue slots and
// the FMA pipe -- not latency -- is the limit.  Kinds:
//   GDT_PROBE_FFMA   fma.rn.f32          2 FLOP per lane-op
//   GDT_PROBE_FFMA2  fma.rn.f32x2 (sm_100 packed FFMA2), 4 FLOP per lane-op
//   GDT_PROBE_DFMA   fma.rn.f64          2 FLOP per lane-op
// FLOP per launch = blocks * 256 * iters * UNROLL * CHAINS * (2 or 4).
#include "common.cuh"

namespace gdt {
namespace {

constexpr int kChains = 8;
constexpr int kUnroll = 16;

__global__ void __launch_bounds__(256) ffma_probe(float *sink, int64_t iters, float seed) {
    float a[kChains];
#pragma unroll
    for (int q = 0; q < kChains; ++q) a[q] = seed + threadIdx.x * 1e-7f + q;
    const float m = 0.9999999f, c = 1e-7f;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int q = 0; q < kChains; ++q) a[q] = fmaf(a[q], m, c);
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < kChains; ++q) s += a[q];
    if (s == 12345.678f) sink[0] = s;  // never true; keeps the chains alive
}

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long ra, rb, rc, rd;
    ra = *reinterpret_cast<unsigned long long *>(&a);
    rb = *reinterpret_cast<unsigned long long *>(&b);
    rc = *reinterpret_cast<unsigned long long *>(&c);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
    return *reinterpret_cast<float2 *>(&rd);
}

__global__ void __launch_bounds__(256) ffma2_probe(float *sink, int64_t iters, float seed) {
    float2 a[kChains];
#pragma unroll
    for (int q = 0; q < kChains; ++q)
        a[q] = make_float2(seed + threadIdx.x * 1e-7f + q, seed - threadIdx.x * 1e-7f - q);
    const float2 m = make_float2(0.9999999f, 0.9999998f), c = make_float2(1e-7f, 2e-7f);
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int q = 0; q < kChains; ++q) a[q] = fma2(a[q], m, c);
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < kChains; ++q) s += a[q].x + a[q].y;
    if (s == 12345.678f) sink[0] = s;
}

__global__ void __launch_bounds__(256) dfma_probe(float *sink, int64_t iters, double seed) {
    double a[kChains];
#pragma unroll
    for (int q = 0; q < kChains; ++q) a[q] = seed + threadIdx.x * 1e-9 + q;
    const double m = 0.999999999, c = 1e-9;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int q = 0; q < kChains; ++q) a[q] = fma(a[q], m, c);
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kChains; ++q) s += a[q];
    if (s == 12345.678) sink[0] = (float)s;
}

// one warp, one dependent chain of DADDs over shared-memory operands (the
// loop shape of chain_sum in primal.cu: 8 operands loaded ahead of 8 adds)
__global__ void __launch_bounds__(32) dadd_chain_probe(long long *cycles, int64_t adds, double seed) {
    __shared__ double ops[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) ops[i] = seed * (1.0 + i * 1e-9);
    __syncwarp();
    double acc = 0.0;
    const long long t0 = clock64();
    for (int64_t j = 0; j + 8 <= adds; j += 8) {
        const double2 *q = reinterpret_cast<const double2 *>(ops + (j & 1016));
        const double2 c0 = q[0], c1 = q[1], c2 = q[2], c3 = q[3];
        acc = __dadd_rn(acc, c0.x);
        acc = __dadd_rn(acc, c0.y);
        acc = __dadd_rn(acc, c1.x);
        acc = __dadd_rn(acc, c1.y);
        acc = __dadd_rn(acc, c2.x);
        acc = __dadd_rn(acc, c2.y);
        acc = __dadd_rn(acc, c3.x);
        acc = __dadd_rn(acc, c3.y);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        cycles[0] = t1 - t0;
        if (acc == 12345.678) cycles[0] = 0;  // keeps the chain alive
    }
}

}  // namespace
}  // namespace gdt

extern "C" int gdt_probe_dadd_chain(int64_t adds, long long *cycles, void *stream) {
    GDT_CHECK_ARG(adds >= 8 && cycles != nullptr, "gdt_probe_dadd_chain: bad arguments");
    gdt::dadd_chain_probe<<<1, 32, 0, gdt::as_stream(stream)>>>(cycles, adds, 1.0);
    return gdt::cuda_status("gdt_probe_dadd_chain");
}

extern "C" int gdt_probe_peak(int kind, int64_t blocks, int64_t iters, float *sink,
                              void *stream) {
    GDT_CHECK_ARG(blocks >= 1 && iters >= 1, "gdt_probe_peak: bad sizes");
    cudaStream_t st = gdt::as_stream(stream);
    switch (kind) {
        case GDT_PROBE_FFMA: gdt::ffma_probe<<<(unsigned)blocks, 256, 0, st>>>(sink, iters, 1.0f); break;
        case GDT_PROBE_FFMA2: gdt::ffma2_probe<<<(unsigned)blocks, 256, 0, st>>>(sink, iters, 1.0f); break;
        case GDT_PROBE_DFMA: gdt::dfma_probe<<<(unsigned)blocks, 256, 0, st>>>(sink, iters, 1.0); break;
        default: GDT_CHECK_ARG(false, "gdt_probe_peak: unknown kind");
    }
    return gdt::cuda_status("gdt_probe_peak");
}

extern "C" int64_t gdt_probe_flops(int kind, int64_t blocks, int64_t iters) {
    const int64_t per = kind == GDT_PROBE_FFMA2 ? 4 : 2;
    return blocks * 256 * iters * gdt::kUnroll * gdt::kChains * per;
}

extern "C" int gdt_probe_fp32(int64_t blocks, int64_t iters, float *sink, void *stream) {
    return gdt_probe_peak(GDT_PROBE_FFMA, blocks, iters, sink, stream);
}
