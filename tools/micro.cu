// Per-pipe issue-rate microbenchmarks on the B200 (SURVEY §2.5 K8,
// §8(d)-D3 "confirm with microbenchmarks").  Each kernel runs long chains of ONE SASS
// instruction class (checked with cuobjdump -sass, see tools/micro.py), 8 independent
// chains per thread, 2 CTAs x 512 threads per SM (32 warps), every CTA co-resident, and
// reports lane-operations per SM clock: total lane-ops / 148 / (max CTA clock64 span).
// The "eo_sign_step" kernel is the K2 sign-uniform step itself (maps.cuh eo_g_biased +
// the update, V = 32 cells per lane, one shuffle per step) on register data: the
// compute-only ceiling of the headline kernel's instruction mix.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I csrc -I include
//        tools/micro.cu -o tools/micro     (tools/micro.py does this)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "fqnm_internal.h"
#include "maps.cuh"

using namespace fqnm;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;           // independent chains per thread

struct Span { unsigned long long t0, t1; };

__device__ __forceinline__ void span_begin(unsigned long long& t0) { t0 = clock64(); }
__device__ __forceinline__ void span_end(Span* s, unsigned long long t0)
{
    __syncthreads();
    if (threadIdx.x == 0) { s[blockIdx.x].t0 = t0; s[blockIdx.x].t1 = clock64(); }
}

// ---- single-class kernels (8 ops per iteration per chain group) ----
#define CHAIN_KERNEL(NAME, TYPE, INIT, OP)                                              \
__global__ void __launch_bounds__(512, 2) NAME(TYPE* out, Span* sp, TYPE a, TYPE b)    \
{                                                                                       \
    unsigned long long t0; __syncthreads(); span_begin(t0);                             \
    TYPE x[CH];                                                                          \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) x[c] = INIT;                         \
    for (int i = 0; i < ITERS; ++i) {                                                   \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) { OP; }                          \
    }                                                                                   \
    TYPE s = x[0];                                                                       \
    _Pragma("unroll") for (int c = 1; c < CH; ++c) s = s + x[c];                        \
    if (s == a) out[threadIdx.x] = s;                                                   \
    span_end(sp, t0);                                                                   \
}

CHAIN_KERNEL(k_iadd3, int32_t, (int32_t)(threadIdx.x + c),
             asm volatile("add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(x[c]) : "r"(a), "r"(b)))
CHAIN_KERNEL(k_lop3, int32_t, (int32_t)(threadIdx.x + c),
             asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b)))
CHAIN_KERNEL(k_imad, int32_t, (int32_t)(threadIdx.x + c),
             asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b)))
CHAIN_KERNEL(k_imad_hi, int32_t, (int32_t)(threadIdx.x + c),
             asm volatile("mad.hi.s32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b)))
CHAIN_KERNEL(k_ffma, float, (float)(threadIdx.x + c),
             asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(a), "f"(b)))
CHAIN_KERNEL(k_dfma, double, (double)(threadIdx.x + c),
             asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b)))
CHAIN_KERNEL(k_i2fp, int32_t, (int32_t)(threadIdx.x + c),
             { float t; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(t) : "r"(x[c]));
               x[c] = __float_as_int(t) >> 8; })
CHAIN_KERNEL(k_lea_hi, int32_t, (int32_t)(threadIdx.x + c),
             { int32_t t = x[c] >> 31; asm volatile("add.s32 %0, %0, %1;" : "+r"(x[c]) : "r"(t)); x[c] ^= a; })

CHAIN_KERNEL(k_dadd, double, (double)(threadIdx.x + c),
             asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[c]) : "d"(a)))
CHAIN_KERNEL(k_imad_wide, long long, (long long)(threadIdx.x + c),
             { int lo = (int)x[c]; asm volatile("mad.wide.s32 %0, %1, %1, %2;" : "=l"(x[c]) : "r"(lo), "l"((long long)b)); })

// ---- DFMA + DADD alternating (independent chains): the float64 half of the EO map ----
__global__ void __launch_bounds__(512, 2) k_dfma_dadd(double* out, Span* sp, double a, double b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    double x[CH], y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = threadIdx.x - c; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
            asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(y[c]) : "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + y[c];
    if (s == 123456789.0) out[threadIdx.x] = s;
    span_end(sp, t0);
}

// ---- IMAD.WIDE + DFMA alternating (independent chains): do they share a pipe? ----
__global__ void __launch_bounds__(512, 2) k_imadwide_dfma(double* out, Span* sp, double a, double b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    double x[CH]; long long y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = threadIdx.x - c; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
            { int lo = (int)y[c]; asm volatile("mad.wide.s32 %0, %1, %1, %2;" : "=l"(y[c]) : "r"(lo), "l"(5ll)); }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + (double)y[c];
    if (s == 123456789.0) out[threadIdx.x] = s;
    span_end(sp, t0);
}

// ---- IMAD.WIDE + IMAD alternating ----
__global__ void __launch_bounds__(512, 2) k_imadwide_imad(int32_t* out, Span* sp, int32_t a, int32_t b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    int32_t x[CH]; long long y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = threadIdx.x - c; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            { int lo = (int)y[c]; asm volatile("mad.wide.s32 %0, %1, %1, %2;" : "=l"(y[c]) : "r"(lo), "l"(5ll)); }
        }
    }
    long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + y[c];
    if (s == 123456789) out[threadIdx.x] = (int32_t)s;
    span_end(sp, t0);
}

// ---- groups of independent instructions: MASK bit 0 DFMA, 1 DADD, 2 IMAD.WIDE, 3 IADD3, 4 IMAD ----
template <int MASK>
__global__ void __launch_bounds__(512, 2) k_group(double* out, Span* sp, double a, double b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    double x[CH], z[CH]; long long y[CH]; int w[CH], v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; z[c] = threadIdx.x * 3 + c; y[c] = threadIdx.x - c; w[c] = c; v[c] = c + 1; }
    const int ia = (int)a + 3, ib = (int)b + 5;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MASK & 1) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
            if (MASK & 2) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(z[c]) : "d"(b));
            if (MASK & 4) { int lo = (int)y[c]; asm volatile("mad.wide.s32 %0, %1, %1, %2;" : "=l"(y[c]) : "r"(lo), "l"(5ll)); }
            if (MASK & 8) asm volatile("add.s32 %0, %0, %1;" : "+r"(w[c]) : "r"(ia));
            if (MASK & 16) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(ia), "r"(ib));
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + z[c] + (double)y[c] + w[c] + v[c];
    if (s == 123456789.0) out[threadIdx.x] = s;
    span_end(sp, t0);
}

// ---- the four instructions of the float64 step with selectable dependences between them:
// MODE bit 0: DFMA reads the IMAD.WIDE result, bit 1: DADD reads the DFMA result,
// bit 2: IADD reads the low word of the DADD result (else each type has its own chain) ----
template <int MODE>
__global__ void __launch_bounds__(512, 2) k_dep(double* out, Span* sp, double a, double b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    double x[CH], z[CH]; long long y[CH]; int w[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; z[c] = threadIdx.x * 3 + c; y[c] = threadIdx.x - c; w[c] = c + threadIdx.x; }
    const int ia = (int)a + 3;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            asm volatile("mad.wide.s32 %0, %1, %1, %2;" : "=l"(y[c]) : "r"(w[c]), "l"(0x4330000000000000ll));
            if (MODE & 1) asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(x[c]) : "d"(__longlong_as_double(y[c])), "d"(a), "d"(b));
            else asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
            if (MODE & 2) asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(z[c]) : "d"(x[c]), "d"(6755399441055744.0));
            else asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(z[c]) : "d"(b));
            if (MODE & 4) asm volatile("add.s32 %0, %0, %1;" : "+r"(w[c]) : "r"(__double2loint(z[c])));
            else asm volatile("add.s32 %0, %0, %1;" : "+r"(w[c]) : "r"(ia));
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + z[c] + (double)y[c] + w[c];
    if (s == 123456789.0) out[threadIdx.x] = s;
    span_end(sp, t0);
}

// ---- mixed streams: ALU + FMA-pipe interleaved 1:1 (independent chains) ----
__global__ void __launch_bounds__(512, 2) k_mixed_alu_fma(int32_t* out, Span* sp, int32_t a, int32_t b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    int32_t x[CH], y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = threadIdx.x - c; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(a), "r"(b));
        }
    }
    int32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] ^ y[c];
    if (s == 123456789) out[threadIdx.x] = s;
    span_end(sp, t0);
}

__global__ void __launch_bounds__(512, 2) k_shfl(int32_t* out, Span* sp, int32_t a, int32_t b)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    int32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __shfl_up_sync(0xffffffffu, x[c], 1);
    }
    int32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 123456789) out[threadIdx.x] = s;
    span_end(sp, t0);
}

// ---- the K2 sign-uniform step on register data (V = 32, 256-thread CTAs, 2 per SM,
// 128 registers: the headline kernel's configuration without its loads/stores) ----
constexpr int SV = 32;
constexpr int SSTEPS = 256;
__global__ void __launch_bounds__(256, 2) k_eo_sign_step(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[SV];
#pragma unroll
    for (int j = 0; j < SV; ++j) q[j] = 100000 + ((seed + 37 * j + 11 * (int)threadIdx.x) & 4095);
    for (int s = 0; s < SSTEPS; ++s) {
        const int32_t glast = eo_g_biased<R_EO_P1, true>(q[SV - 1], r);
        int32_t gp = __shfl_up_sync(0xffffffffu, glast, 1);
#pragma unroll
        for (int j = 0; j + 1 < SV; ++j) {                 // as kernels_scalar.cu one_step
            const int32_t gj = eo_g_biased<R_EO_P1, false>(q[j], r);
            q[j] = q[j] + gp - gj;
            gp = gj;
        }
        q[SV - 1] = q[SV - 1] + gp - glast;
        if (lane == 0) q[0] = 100000;        // keep the window's data positive and bounded
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SV; ++j) acc ^= q[j];
    if (acc == 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

// ---- the K2 sign-uniform step with the float64 map (IMAD.WIDE, DFMA, DADD, IADD3) ----
__global__ void __launch_bounds__(256, 2) k_eo_dp_step(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[SV];
#pragma unroll
    for (int j = 0; j < SV; ++j) q[j] = 100000 + ((seed + 37 * j + 11 * (int)threadIdx.x) & 4095);
    for (int s = 0; s < SSTEPS; ++s) {
        const int32_t glast = eo_g_dp(q[SV - 1], r);
        int32_t gp = __shfl_up_sync(0xffffffffu, glast, 1);
#pragma unroll
        for (int j = 0; j + 1 < SV; ++j) {
            const int32_t gj = eo_g_dp(q[j], r);
            q[j] = q[j] + gp - gj;
            gp = gj;
        }
        q[SV - 1] = q[SV - 1] + gp - glast;
        if (lane == 0) q[0] = 100000;
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SV; ++j) acc ^= q[j];
    if (acc == 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

// ---- the float64 step at other occupancies / with the offset in an ordinary register ----
template <int MINB, int NV, bool REGOFF>
__global__ void __launch_bounds__(256, MINB) k_eo_dp_occ(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) q[j] = 100000 + ((seed + 37 * j + 11 * (int)threadIdx.x) & 4095);
    long long xo = r.eo_xoff;
    double dinv = r.eo_dinv, dc1 = r.eo_dc1;
    if (REGOFF) { xo += threadIdx.x >> 20; asm volatile("" : "+l"(xo), "+d"(dinv), "+d"(dc1)); }
    auto gdp = [&](int32_t x) {
        const long long X = (long long)x * (long long)x + xo;
        return __double2loint(__dadd_rn(__fma_rn(__longlong_as_double(X), dinv, dc1), 6755399441055744.0));
    };
    for (int s = 0; s < SSTEPS; ++s) {
        const int32_t glast = gdp(q[NV - 1]);
        int32_t gp = __shfl_up_sync(0xffffffffu, glast, 1);
#pragma unroll
        for (int j = 0; j + 1 < NV; ++j) {
            const int32_t gj = gdp(q[j]);
            q[j] = q[j] + gp - gj;
            gp = gj;
        }
        q[NV - 1] = q[NV - 1] + gp - glast;
        if (lane == 0) q[0] = 100000;
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < NV; ++j) acc ^= q[j];
    if (acc == 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

// ---- float64 step variants of how the FP64 result reaches the integer update:
// MODE 1: through an IMAD (FMA-heavy pipe) copy; MODE 2: the update itself as two IMADs;
// MODE 3: differences taken in float64 (DADD of the two magic-biased values), one conversion ----
template <int MODE>
__global__ void __launch_bounds__(256, 2) k_eo_dp_route(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[SV];
#pragma unroll
    for (int j = 0; j < SV; ++j) q[j] = 100000 + ((seed + 37 * j + 11 * (int)threadIdx.x) & 4095);
    const int one = r.one, mone = r.mone;
    auto tdp = [&](int32_t x) {
        const long long X = (long long)x * (long long)x + r.eo_xoff;
        return __dadd_rn(__fma_rn(__longlong_as_double(X), r.eo_dinv, r.eo_dc1), 6755399441055744.0);
    };
    for (int s = 0; s < SSTEPS; ++s) {
        const double tl = tdp(q[SV - 1]);
        const int32_t glast = __double2loint(tl);
        int32_t gp = __shfl_up_sync(0xffffffffu, glast, 1);
        double tp = __hiloint2double(0x43380000, gp);
#pragma unroll
        for (int j = 0; j + 1 < SV; ++j) {
            const double t = tdp(q[j]);
            if (MODE == 1) {
                int32_t gj;
                asm volatile("mad.lo.s32 %0, %1, %2, 0;" : "=r"(gj) : "r"(__double2loint(t)), "r"(one));
                q[j] = q[j] + gp - gj;
                gp = gj;
            } else if (MODE == 2) {
                const int32_t gj = __double2loint(t);
                int32_t u;
                asm volatile("mad.lo.s32 %0, %1, %2, %3;" : "=r"(u) : "r"(gj), "r"(mone), "r"(q[j]));
                asm volatile("mad.lo.s32 %0, %1, %2, %3;" : "=r"(q[j]) : "r"(gp), "r"(one), "r"(u));
                gp = gj;
            } else {
                // d = tp - t is exact (both 1.5 2^52 + g); q + d in float64 needs q as double: instead
                // take the low word of (tp - t) + magic
                const double d = __dadd_rn(__dadd_rn(tp, -t), 6755399441055744.0);
                q[j] = q[j] + __double2loint(d);
                tp = t;
            }
        }
        q[SV - 1] = q[SV - 1] + (MODE == 3 ? __double2loint(tp) : gp) - glast;
        if (lane == 0) q[0] = 100000;
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SV; ++j) acc ^= q[j];
    if (acc == 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

// ---- the float64 step in batches of B cells (producer -> consumer distance B) ----
template <int B>
__global__ void __launch_bounds__(256, 2) k_eo_dp_batch(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[SV];
#pragma unroll
    for (int j = 0; j < SV; ++j) q[j] = 100000 + ((seed + 37 * j + 11 * (int)threadIdx.x) & 4095);
    for (int s = 0; s < SSTEPS; ++s) {
        const int32_t glast = eo_g_dp(q[SV - 1], r);
        int32_t gp = __shfl_up_sync(0xffffffffu, glast, 1);
#pragma unroll
        for (int j0 = 0; j0 + 1 < SV; j0 += B) {
            double X[B], t[B];
#pragma unroll
            for (int b = 0; b < B; ++b)
                if (j0 + b + 1 < SV)
                    X[b] = __longlong_as_double((long long)q[j0 + b] * (long long)q[j0 + b] + r.eo_xoff);
#pragma unroll
            for (int b = 0; b < B; ++b)
                if (j0 + b + 1 < SV) t[b] = __fma_rn(X[b], r.eo_dinv, r.eo_dc1);
#pragma unroll
            for (int b = 0; b < B; ++b)
                if (j0 + b + 1 < SV) t[b] = __dadd_rn(t[b], 6755399441055744.0);
#pragma unroll
            for (int b = 0; b < B; ++b)
                if (j0 + b + 1 < SV) {
                    const int32_t gj = __double2loint(t[b]);
                    q[j0 + b] = q[j0 + b] + gp - gj;
                    gp = gj;
                }
        }
        q[SV - 1] = q[SV - 1] + gp - glast;
        if (lane == 0) q[0] = 100000;
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SV; ++j) acc ^= q[j];
    if (acc == 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

// ---- the K2 LIN kappa = 1/2 step on register data (cfg3's mix: LEA.HI + SHF + 2 IMAD) ----
__global__ void __launch_bounds__(256, 2) k_lin_half_step(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[SV];
#pragma unroll
    for (int j = 0; j < SV; ++j) q[j] = ((seed + 37 * j + 11 * (int)threadIdx.x) & 8191) - 4096;
    for (int s = 0; s < SSTEPS; ++s) {
        int32_t h[SV], p[SV];
#pragma unroll
        for (int j = 0; j < SV; ++j) {
            h[j] = q[j] / 2;
            p[j] = h[j] * r.mone + q[j];
        }
        const int32_t pl = __shfl_up_sync(0xffffffffu, p[SV - 1], 1);
        q[0] = pl * r.one + h[0];
#pragma unroll
        for (int j = 1; j < SV; ++j) q[j] = p[j - 1] * r.one + h[j];
        if (lane == 0) q[0] = 777;
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SV; ++j) acc ^= q[j];
    if (acc == seed + 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

// ---- EO sign-step variants (cells per clock; exploration of the instruction mix) ----
// CONV: 0 I2FP, 1 IMAD + FADD, 2 alternate; ORD: 0 v = q*q + (bits*nQ + c6),
// 1 v = bits*nQ + (q*q + c6) (the q*q IMAD off the float chain's critical path)
template <int CONV, int ORD>
__device__ __forceinline__ int32_t g_var(int32_t q, const DevRule& r, bool odd)
{
    float qf;
    if (CONV == 0 || (CONV == 2 && !odd)) qf = __int2float_rn(q);
    else qf = __int_as_float(imad(q, r.one, 0x4B400000)) - 12582912.0f;
    const float sq = __fmul_rn(qf, qf);
    const float t = __fmaf_rn(sq, r.eo_cf, 12582913.0f);
    const int32_t bits = __float_as_int(t);
    int32_t v;
    if (ORD == 0) v = imad(q, q, imad(bits, r.eo_nQ, r.eo_c6));
    else v = imad(bits, r.eo_nQ, imad(q, q, r.eo_c6));
    return bits + (v >> 31);
}

template <int CONV, int ORD, int MINB>
__global__ void __launch_bounds__(256, MINB) k_eo_var(int32_t* out, Span* sp, DevRule r, int32_t seed)
{
    unsigned long long t0; __syncthreads(); span_begin(t0);
    const int lane = threadIdx.x & 31;
    int32_t q[SV];
#pragma unroll
    for (int j = 0; j < SV; ++j) q[j] = 100000 + ((seed + 37 * j + 11 * (int)threadIdx.x) & 4095);
    for (int s = 0; s < SSTEPS; ++s) {
        const int32_t glast = g_var<CONV, ORD>(q[SV - 1], r, true);
        int32_t gp = __shfl_up_sync(0xffffffffu, glast, 1);
#pragma unroll
        for (int j = 0; j + 1 < SV; ++j) {
            const int32_t gj = g_var<CONV, ORD>(q[j], r, (j & 1) != 0);
            q[j] = q[j] + gp - gj;
            gp = gj;
        }
        q[SV - 1] = q[SV - 1] + gp - glast;
        if (lane == 0) q[0] = 100000;
    }
    int32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SV; ++j) acc ^= q[j];
    if (acc == seed + 123456789) out[threadIdx.x] = acc;
    span_end(sp, t0);
}

int main(int argc, char** argv)
{
    const int sms = 148;
    Span* sp;
    void* out;
    CK(cudaMalloc(&sp, sms * 4 * sizeof(Span)));
    CK(cudaMalloc(&out, 4096 * 8));
    std::vector<Span> h(sms * 4);
    auto measure = [&](const char* name, const char* sass, int blocks_per_sm, int threads,
                       double lane_ops_per_thread, auto launch) -> int {
        const int blocks = sms * blocks_per_sm;
        double best = 0, best_ns = 0;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            launch(blocks, threads);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            CK(cudaMemcpy(h.data(), sp, blocks * sizeof(Span), cudaMemcpyDeviceToHost));
            unsigned long long span = 0;
            for (int b = 0; b < blocks; ++b) span = h[b].t1 - h[b].t0 > span ? h[b].t1 - h[b].t0 : span;
            const double ops_sm = lane_ops_per_thread * threads * blocks_per_sm;
            const double rate = ops_sm / (double)span;
            if (rate > best) { best = rate; best_ns = ms * 1e6; }
            cudaEventDestroy(e0); cudaEventDestroy(e1);
        }
        printf("{\"name\": \"%s\", \"sass\": \"%s\", \"lane_ops_per_clk_per_sm\": %.3f, "
               "\"warp_instr_per_clk_per_smsp\": %.4f, \"kernel_ns\": %.0f, "
               "\"lane_ops_per_s\": %.6e}\n",
               name, sass, best, best / 128.0, best_ns,
               lane_ops_per_thread * threads * blocks / (best_ns * 1e-9));
        return 0;
    };
    const double n1 = (double)ITERS * CH;
    int32_t a = 3, b = 5;
#define L1(K, T, A, B) [&](int g, int t) { K<<<g, t>>>((T*)out, sp, (T)(A), (T)(B)); }
    measure("iadd3", "IADD3", 2, 512, n1, L1(k_iadd3, int32_t, a, b));
    measure("lop3", "LOP3", 2, 512, n1, L1(k_lop3, int32_t, a, b));
    measure("imad", "IMAD", 2, 512, n1, L1(k_imad, int32_t, a, b));
    measure("imad_hi", "IMAD.HI", 2, 512, n1, L1(k_imad_hi, int32_t, a, b));
    measure("ffma", "FFMA", 2, 512, n1, L1(k_ffma, float, 1.0001f, 0.5f));
    measure("dfma", "DFMA", 2, 512, n1, L1(k_dfma, double, 1.0000001, 0.5));
    measure("dadd", "DADD", 2, 512, n1, L1(k_dadd, double, 1.5, 0.5));
    measure("dfma_dadd", "DFMA + DADD interleaved (per op)", 2, 512, 2 * n1, L1(k_dfma_dadd, double, 1.0000001, 0.5));
    measure("imad_wide", "IMAD.WIDE", 2, 512, n1, L1(k_imad_wide, long long, 3, 5));
    measure("imadwide_dfma", "IMAD.WIDE + DFMA interleaved (per op)", 2, 512, 2 * n1, L1(k_imadwide_dfma, double, 1.0000001, 0.5));
    measure("imadwide_imad", "IMAD.WIDE + IMAD interleaved (per op)", 2, 512, 2 * n1, L1(k_imadwide_imad, int32_t, a, b));
#define GRP(M, N, NAME, WHAT) measure(NAME, WHAT " (per op)", 2, 512, N * n1, \
        [&](int g, int t) { k_group<M><<<g, t>>>((double*)out, sp, 1.0000001, 0.5); })
    GRP(7, 3, "grp_dfma_dadd_imadwide", "DFMA + DADD + IMAD.WIDE");
    GRP(11, 3, "grp_dfma_dadd_iadd", "DFMA + DADD + IADD");
    GRP(15, 4, "grp_dfma_dadd_imadwide_iadd", "DFMA + DADD + IMAD.WIDE + IADD");
    GRP(19, 3, "grp_dfma_dadd_imad", "DFMA + DADD + IMAD");
    GRP(9, 2, "grp_dfma_iadd", "DFMA + IADD");
    GRP(13, 3, "grp_dfma_imadwide_iadd", "DFMA + IMAD.WIDE + IADD");
#define DEP(M, NAME) measure(NAME, "IMAD.WIDE, DFMA, DADD, IADD with dependences (mode bits) (per op)", 2, 512, 4 * n1, \
        [&](int g, int t) { k_dep<M><<<g, t>>>((double*)out, sp, 1.0000001, 0.5); })
    DEP(0, "dep0_none"); DEP(1, "dep1_wide_to_dfma"); DEP(2, "dep2_dfma_to_dadd"); DEP(4, "dep4_dadd_to_iadd");
    DEP(3, "dep3"); DEP(6, "dep6"); DEP(7, "dep7_all");
    measure("i2fp_shf", "I2FP + SHF pairs (per op)", 2, 512, 2 * n1, L1(k_i2fp, int32_t, 0, 0));
    measure("lea_hi", "LEA.HI + LOP3 pairs (per op)", 2, 512, 2 * n1, L1(k_lea_hi, int32_t, a, b));
    measure("mixed_alu_fma_int", "LOP3 + IMAD interleaved", 2, 512, 2 * n1, L1(k_mixed_alu_fma, int32_t, a, b));
    measure("shfl", "SHFL.UP", 2, 512, n1, L1(k_shfl, int32_t, a, b));
    DevRule r;
    std::memset(&r, 0, sizeof r);
    const int64_t Q = 1724240;                              // cfg4's kappa = 1/Q
    r.one = 1; r.mone = -1;
    r.eo_cf = (float)(1.0 / (double)Q * (1.0 - 1.0 / 2097152.0));
    r.eo_nQ = (int32_t)(-Q);
    r.eo_c6 = (int32_t)(uint32_t)((uint64_t)Q * 0x4B400001ull - (uint64_t)((Q + 1) / 2));
    // 7 instructions per cell-update (I2FP, FMUL, FFMA, 2 IMAD, LEA.HI, IADD3)
    measure("eo_sign_step", "K2 sign-uniform step, 7 instr/cell", 2, 256, 7.0 * SSTEPS * SV,
            [&](int g, int t) { k_eo_sign_step<<<g, t>>>((int32_t*)out, sp, r, 17); });
    {
        const long double inv = (1.0L / (long double)Q) * (1.0L + ldexpl(1.0L, -46));
        r.eo_dinv = (double)inv;
        r.eo_dc1 = -ldexp(r.eo_dinv, 52);
        r.eo_xoff = (long long)(1023 + 52) << 52;
    }
    // 4 instructions per cell-update (IMAD.WIDE, DFMA, DADD, IADD3)
    measure("eo_dp_step", "K2 sign-uniform step, float64 map, 4 instr/cell", 2, 256, 4.0 * SSTEPS * SV,
            [&](int g, int t) { k_eo_dp_step<<<g, t>>>((int32_t*)out, sp, r, 17); });
#define DPO(MB, NV, RO, NAME) measure(NAME, "float64 step variants (4 instr/cell)", MB, 256, \
        4.0 * SSTEPS * NV, [&](int g, int t) { k_eo_dp_occ<MB, NV, RO><<<g, t>>>((int32_t*)out, sp, r, 17); })
    DPO(2, 32, true, "eo_dp_regoff"); DPO(3, 32, false, "eo_dp_occ3"); DPO(4, 32, false, "eo_dp_occ4");
    DPO(4, 16, false, "eo_dp_occ4_v16"); DPO(8, 16, false, "eo_dp_occ8_v16"); DPO(1, 32, false, "eo_dp_occ1");
#define DPR(M, NI, NAME) measure(NAME, "float64 step, result routing variants (cells x 4)", 2, 256, \
        4.0 * SSTEPS * SV, [&](int g, int t) { k_eo_dp_route<M><<<g, t>>>((int32_t*)out, sp, r, 17); })
    DPR(1, 5, "eo_dp_route_imadcopy"); DPR(2, 5, "eo_dp_route_imadupdate"); DPR(3, 6, "eo_dp_route_f64diff");
#define DPB(BB, NAME) measure(NAME, "float64 step in batches of B cells (4 instr/cell)", 2, 256, \
        4.0 * SSTEPS * SV, [&](int g, int t) { k_eo_dp_batch<BB><<<g, t>>>((int32_t*)out, sp, r, 17); })
    DPB(4, "eo_dp_batch4"); DPB(8, "eo_dp_batch8"); DPB(16, "eo_dp_batch16"); DPB(31, "eo_dp_batch31");
    // EO variants: reported as lane-ops at 7 per cell, i.e. cells/clk x 7 (comparable)
#define EOV(C, O, M, NAME) measure(NAME, "EO sign-step variant (7-op-equivalent cells)", M, 256, \
        7.0 * SSTEPS * SV, [&](int g, int t) { k_eo_var<C, O, M><<<g, t>>>((int32_t*)out, sp, r, 17); })
    EOV(0, 0, 2, "eo_var_conv0_ord0");
    EOV(0, 1, 2, "eo_var_conv0_ord1");
    EOV(1, 0, 2, "eo_var_conv1_ord0");
    EOV(1, 1, 2, "eo_var_conv1_ord1");
    EOV(2, 1, 2, "eo_var_conv2_ord1");
    // 4 instructions per cell-update (LEA.HI, SHF, 2 IMAD)
    measure("lin_half_step", "K2 LIN 1/2 step, 4 instr/cell", 2, 256, 4.0 * SSTEPS * SV,
            [&](int g, int t) { k_lin_half_step<<<g, t>>>((int32_t*)out, sp, r, 17); });
    return 0;
}
