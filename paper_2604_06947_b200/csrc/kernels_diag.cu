// Level-space diagnostics of the quantised state (PAPER.md Supplementary
// Information):
//   c_k = #{i : q_i = k},  p_k = c_k / N,  S = -sum_k p_k log p_k,  N_eff = exp S
//   N_{k'k} = #{i : q^n_i = k and q^{n+1}_i = k'},  M_{k'k} = N_{k'k} / c^n_k
//   rho = max_{k'} |sum_k M_{k'k} - 1|  over the union of the two supports.
// Kernels: a dense level histogram (global atomics), an entropy reduction over
// the histogram, and an open-addressing hash aggregation of (k, k') pairs.
// Also the transfer-operator equivalence checker (Thm P:262-280): one explicit
// step of rule a while rule b is evaluated on every visited interface state.
#include <cstdint>
#include <cuda_runtime.h>

#include "fqnm_internal.h"
#include "maps.cuh"

namespace fqnm {

template <typename T>
__global__ void k_histogram(const T* __restrict__ q, int64_t n, int64_t lo, int64_t L,
                            unsigned int* __restrict__ counts, unsigned long long* __restrict__ outside)
{
    unsigned long long out = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = (int64_t)q[i] - lo;
        if (k >= 0 && k < L) atomicAdd(counts + k, 1u);
        else ++out;
    }
    if (out) atomicAdd(outside, out);
}

// sum_k c_k log c_k (double) and the number of occupied levels
__global__ void k_clogc(const unsigned int* __restrict__ counts, int64_t L, double* __restrict__ acc,
                        unsigned long long* __restrict__ occupied)
{
    double s = 0.0;
    unsigned long long occ = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < L;
         k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned int c = counts[k];
        if (c) {
            s += (double)c * log((double)c);
            ++occ;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        occ += __shfl_xor_sync(0xffffffffu, occ, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, s);
        atomicAdd(occupied, occ);
    }
}

static constexpr unsigned long long EMPTY = 0xffffffffffffffffull;

// aggregate pair keys (k - lo) * L + (k' - lo) into an open-addressing table
template <typename T>
__global__ void k_pairs(const T* __restrict__ q0, const T* __restrict__ q1, int64_t n, int64_t lo,
                        int64_t L, unsigned long long* __restrict__ keys,
                        unsigned int* __restrict__ vals, unsigned long long mask,
                        unsigned long long* __restrict__ overflow)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = (int64_t)q0[i] - lo, b = (int64_t)q1[i] - lo;
        if (a < 0 || a >= L || b < 0 || b >= L) continue;
        const unsigned long long key = (unsigned long long)a * (unsigned long long)L + (unsigned long long)b;
        unsigned long long h = (key * 0x9E3779B97F4A7C15ull) & mask;
        for (unsigned long long probe = 0; probe <= mask; ++probe) {
            const unsigned long long prev = atomicCAS(keys + h, EMPTY, key);
            if (prev == EMPTY || prev == key) {
                atomicAdd(vals + h, 1u);
                break;
            }
            h = (h + 1) & mask;
            if (probe == mask) atomicAdd(overflow, 1ull);
        }
    }
}

// rowsum[k'] += N_{k'k} / c_k over the table; count the non-empty slots
__global__ void k_rowsums(const unsigned long long* __restrict__ keys,
                          const unsigned int* __restrict__ vals, unsigned long long cap, int64_t L,
                          const unsigned int* __restrict__ c0, double* __restrict__ rowsum,
                          unsigned long long* __restrict__ npairs)
{
    unsigned long long np = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        if (key == EMPTY) continue;
        ++np;
        const int64_t a = (int64_t)(key / (unsigned long long)L), b = (int64_t)(key % (unsigned long long)L);
        atomicAdd(rowsum + b, (double)vals[i] / (double)c0[a]);
    }
    if (np) atomicAdd(npairs, np);
}

// rho = max over the union of supports of |rowsum - 1| (as an ordered uint64 of the double)
__global__ void k_defect(const double* __restrict__ rowsum, const unsigned int* __restrict__ c0,
                         const unsigned int* __restrict__ c1, int64_t L,
                         unsigned long long* __restrict__ maxbits)
{
    double m = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < L;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (c0[k] || c1[k]) {
            const double d = fabs(rowsum[k] - 1.0);
            m = d > m ? d : m;
        }
    }
    // non-negative doubles order like their bit patterns
    atomicMax(maxbits, (unsigned long long)__double_as_longlong(m));
}

static int grid_for_diag(int64_t work) { int64_t g = (work + 255) / 256; return (int)(g > 148 * 8 ? 148 * 8 : (g < 1 ? 1 : g)); }

cudaError_t launch_histogram(const void* q, int dtype, int64_t n, int64_t lo, int64_t L,
                             unsigned int* counts, unsigned long long* outside, cudaStream_t st)
{
    const int g = grid_for_diag(n);
    if (dtype == 0) k_histogram<int32_t><<<g, 256, 0, st>>>((const int32_t*)q, n, lo, L, counts, outside);
    else k_histogram<int64_t><<<g, 256, 0, st>>>((const int64_t*)q, n, lo, L, counts, outside);
    return cudaGetLastError();
}

cudaError_t launch_clogc(const unsigned int* counts, int64_t L, double* acc,
                         unsigned long long* occupied, cudaStream_t st)
{
    k_clogc<<<grid_for_diag(L), 256, 0, st>>>(counts, L, acc, occupied);
    return cudaGetLastError();
}

cudaError_t launch_pairs(const void* q0, const void* q1, int dtype, int64_t n, int64_t lo, int64_t L,
                         unsigned long long* keys, unsigned int* vals, unsigned long long cap,
                         unsigned long long* overflow, cudaStream_t st)
{
    const int g = grid_for_diag(n);
    if (dtype == 0)
        k_pairs<int32_t><<<g, 256, 0, st>>>((const int32_t*)q0, (const int32_t*)q1, n, lo, L, keys,
                                            vals, cap - 1, overflow);
    else
        k_pairs<int64_t><<<g, 256, 0, st>>>((const int64_t*)q0, (const int64_t*)q1, n, lo, L, keys,
                                            vals, cap - 1, overflow);
    return cudaGetLastError();
}

cudaError_t launch_rowsums(const unsigned long long* keys, const unsigned int* vals,
                           unsigned long long cap, int64_t L, const unsigned int* c0, double* rowsum,
                           unsigned long long* npairs, cudaStream_t st)
{
    k_rowsums<<<grid_for_diag((int64_t)cap), 256, 0, st>>>(keys, vals, cap, L, c0, rowsum, npairs);
    return cudaGetLastError();
}

cudaError_t launch_defect(const double* rowsum, const unsigned int* c0, const unsigned int* c1,
                          int64_t L, unsigned long long* maxbits, cudaStream_t st)
{
    k_defect<<<grid_for_diag(L), 256, 0, st>>>(rowsum, c0, c1, L, maxbits);
    return cudaGetLastError();
}

// ---- transfer-operator equivalence (Thm P:262-280) -------------------------
__device__ __forceinline__ int32_t transfer_any(int rule, int32_t qL, int32_t qR, const DevRule& r)
{
    switch (rule) {
        case R_LIN_HALF: return transfer_lr<R_LIN_HALF>(qL, qR, r);
        case R_EO_FAST: return transfer_lr<R_EO_FAST>(qL, qR, r);
        case R_EO_P1: return transfer_lr<R_EO_P1>(qL, qR, r);
        case R_LIN_FAST: return transfer_lr<R_LIN_FAST>(qL, qR, r);
        case R_TWOPOINT: return transfer_lr<R_TWOPOINT>(qL, qR, r);
        case R_TP_FAST: return transfer_lr<R_TP_FAST>(qL, qR, r);
        default: return transfer_lr<R_GENERIC>(qL, qR, r);
    }
}

// interfaces t = 0 .. nI-1: periodic nI = n, interface t + 1/2 between cells t and
// (t+1) mod n; transmissive nI = n + 1, interface t - 1/2 between t-1 and t (ghost copies)
__global__ void k_equiv_transfer(const int32_t* __restrict__ q, int32_t* __restrict__ T, int64_t n,
                                 int bmode, DevRule ra, int rule_a, DevRule rb, int rule_b,
                                 int64_t step, unsigned long long* __restrict__ counters,
                                 unsigned long long* __restrict__ keys,
                                 unsigned int* __restrict__ vals, unsigned long long mask,
                                 int64_t lo, int64_t L)
{
    const int64_t nI = bmode == BM_PERIODIC ? n : n + 1;
    unsigned long long mism = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nI;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t iL, iR;
        if (bmode == BM_PERIODIC) { iL = t; iR = (t + 1 == n) ? 0 : t + 1; }
        else { iL = t == 0 ? 0 : t - 1; iR = t == n ? n - 1 : t; }
        const int32_t qL = q[iL], qR = q[iR];
        const int32_t Ta = transfer_any(rule_a, qL, qR, ra);
        const int32_t Tb = transfer_any(rule_b, qL, qR, rb);
        T[t] = Ta;
        const bool bad = Ta != Tb;
        mism += bad;
        if (mask) {
            const int64_t a = (int64_t)qL - lo, b = (int64_t)qR - lo;
            if (a < 0 || a >= L || b < 0 || b >= L) {
                atomicAdd(counters + 2, 1ull);
            } else {
                const unsigned long long key = (unsigned long long)a * (unsigned long long)L +
                                               (unsigned long long)b;
                unsigned long long h = (key * 0x9E3779B97F4A7C15ull) & mask;
                bool done = false;
                for (unsigned long long probe = 0; probe <= mask; ++probe) {
                    const unsigned long long prev = atomicCAS(keys + h, EMPTY, key);
                    if (prev == EMPTY || prev == key) {
                        atomicOr(vals + h, bad ? 3u : 1u);
                        done = true;
                        break;
                    }
                    h = (h + 1) & mask;
                }
                if (!done) atomicAdd(counters + 2, 1ull);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mism += __shfl_xor_sync(0xffffffffu, mism, o);
    if ((threadIdx.x & 31) == 0 && mism) {
        atomicAdd(counters, mism);
        atomicMin(counters + 1, (unsigned long long)step);
    }
}

// q'_i = q_i - (T_{i+1/2} - T_{i-1/2})  (P:86-89 with the transfer of rule a)
__global__ void k_equiv_update(const int32_t* __restrict__ q, const int32_t* __restrict__ T,
                               int32_t* __restrict__ qn, int64_t n, int bmode)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t Tr = bmode == BM_PERIODIC ? T[i] : T[i + 1];
        const int32_t Tl = bmode == BM_PERIODIC ? T[i == 0 ? n - 1 : i - 1] : T[i];
        qn[i] = q[i] - (Tr - Tl);
    }
}

__global__ void k_equiv_count(const unsigned long long* __restrict__ keys,
                              const unsigned int* __restrict__ vals, unsigned long long cap,
                              unsigned long long* __restrict__ out2)
{
    unsigned long long v = 0, m = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        if (keys[i] != EMPTY) {
            ++v;
            m += (vals[i] >> 1) & 1u;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out2, v);
        atomicAdd(out2 + 1, m);
    }
}

cudaError_t launch_equiv_step(const int32_t* q, int32_t* qn, int32_t* T, int64_t n, int bmode,
                              const DevRule& ra, int rule_a, const DevRule& rb, int rule_b,
                              int64_t step, unsigned long long* counters, unsigned long long* keys,
                              unsigned int* vals, unsigned long long mask, int64_t lo, int64_t L,
                              cudaStream_t st)
{
    k_equiv_transfer<<<grid_for_diag(n + 1), 256, 0, st>>>(q, T, n, bmode, ra, rule_a, rb, rule_b,
                                                           step, counters, keys, vals, mask, lo, L);
    k_equiv_update<<<grid_for_diag(n), 256, 0, st>>>(q, T, qn, n, bmode);
    return cudaGetLastError();
}

cudaError_t launch_equiv_count(const unsigned long long* keys, const unsigned int* vals,
                               unsigned long long cap, unsigned long long* out2, cudaStream_t st)
{
    k_equiv_count<<<grid_for_diag((int64_t)cap), 256, 0, st>>>(keys, vals, cap, out2);
    return cudaGetLastError();
}

}  // namespace fqnm
