// K9: 2D directional composition, streaming (Thm formal Cartesian extension,
// PAPER.md P:364-401, Eq. nd_transfer_rule with d = 2):
//   q'_{i,j} = q - (F^x_{i+1/2,j} - F^x_{i-1/2,j}) - (F^y_{i,j+1/2} - F^y_{i,j-1/2}),
//   F^x_{i+1/2,j} = phi+_x(q_{i,j}) + phi-_x(q_{i+1,j})   (and likewise in y).
// One step per launch, one warp per (x strip, y chunk), no shared memory and no
// barriers: a warp loads 128 consecutive cells of a row (4 per lane, int2 x 2), of
// which the outer 2 on each side are halo (strip stride 124 cells), and marches down
// its chunk of rows.  x neighbours' maps come from the lane's own registers and warp
// shuffles, y neighbours' maps from the rows above and below kept in registers; every
// loaded cell's maps are evaluated once.  Rows stream through a per-warp shared-memory
// ring, 6 rows in flight per lane (cp.async), and the loop is unrolled so the row
// rotation needs no register moves.
// HBM traffic: one read and one write of the state per step (8 B per cell-update),
// 3.1 % redundant halo columns.  Indices are 32-bit (nx * ny < 2^31).
#include <cstdint>
#include <cuda_runtime.h>

#include "fqnm_internal.h"
#include "maps.cuh"

namespace fqnm {

static constexpr unsigned FULL2 = 0xffffffffu;
// resident CTAs per SM asked of ptxas (variant sweeps only): unset = __launch_bounds__(256)
// with no minimum, which measured fastest -- a minimum of 1 alone changes the register
// allocation of the k = 2 kernel and costs 23 % (8192^2 EO 892 -> 687 GCUPS), 3 spills
#if defined(FQNM_K9_MINB1)
#define K9_LB1 __launch_bounds__(256, FQNM_K9_MINB1)
#else
#define K9_LB1 __launch_bounds__(256)
#endif
// k = 2 kernel: a minimum of 2 for the EO rules (8192^2 EO 894 -> 920 GCUPS; linear
// 871 -> 864 with it, so none there; a minimum of 0 is the same as none)
template <int RULE>
constexpr int k9_minb2() { return (RULE == R_EO_P1 || RULE == R_EO_FAST) ? 2 : 0; }
#if defined(FQNM_K9_MINB2)
#define K9_LB2 __launch_bounds__(256, FQNM_K9_MINB2)
#else
#define K9_LB2 __launch_bounds__(256, k9_minb2<RULE>())
#endif
#ifndef FQNM_K9_V
#define FQNM_K9_V 4
#endif
static constexpr int K9_V = FQNM_K9_V;          // x cells per lane (even)
static constexpr int K9_W = 32 * K9_V;          // loaded strip width
static constexpr int K9_H = 2;                  // halo columns per side
static constexpr int K9_S = K9_W - 2 * K9_H;    // strip stride (stored columns)
static constexpr int K9_LOOK = 6;               // rows in flight per lane (cp.async ring)

__device__ __forceinline__ int wrap2(int i, int n, int bmode)
{
    if (bmode == BM_PERIODIC) { i %= n; return i < 0 ? i + n : i; }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);            // transmissive ghost copy
}

__device__ __forceinline__ int wrap_row(int r, int n, int bmode)
{
    if (bmode == BM_PERIODIC) return r < 0 ? r + n : (r >= n ? r - n : r);
    return r < 0 ? 0 : (r >= n ? n - 1 : r);
}

// One row of a lane: the state and its maps.  SAME (one rule for x and y): the maps
// are kept as g = phi+ + phi- (EO P = 1: biased by a constant, see maps.cuh eo_gm_p1),
// m = phi- and pb = g - m = phi+ (+ bias); the update
//   q' = q + (p_l + m_c) - (p_c + m_r) + (p_d + m_c) - (p_c + m_u)
//      = q + pb_l + pb_d - m_r - m_u + 2 (2 m_c - g_c)
// is free of the bias (+2 - 2 in the biased terms) and takes 5 operations per cell.
// The (g, m, pb) form is used for the EO rules with one rule for both directions
// (measured faster there); the linear and generic rules keep (phi+, phi-) per direction.
// Per-warp row ring in shared memory: lane l's V cells of a row as V/2 int2 slots at
// [h][l] (conflict-free 8-byte accesses), filled by the lane itself with cp.async.
struct K9Ring {
    unsigned base;                                  // this lane's slot 0 of stage 0
    static constexpr unsigned HSTRIDE = 32 * 8;     // bytes between the int2 slots of a lane
    static constexpr unsigned STAGE = (K9_V / 2) * HSTRIDE * (256 / 32);
    __device__ __forceinline__ unsigned at(int stg, int h) const { return base + stg * STAGE + h * HSTRIDE; }
    // copy the lane's cells of `row` (fast: 8-byte pieces at xl; else scalar through xo)
    __device__ __forceinline__ void issue(int stg, const int32_t* row, bool vec, int xl,
                                          const int (&xo)[K9_V]) const
    {
        if (vec) {
#pragma unroll
            for (int h = 0; h < K9_V / 2; ++h)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(at(stg, h)), "l"(row + xl + 2 * h) : "memory");
        } else {
#pragma unroll
            for (int j = 0; j < K9_V; ++j)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(at(stg, j / 2) + 4 * (j & 1)), "l"(row + xo[j]) : "memory");
        }
    }
    __device__ __forceinline__ void read(int stg, int32_t (&v)[K9_V]) const
    {
#pragma unroll
        for (int h = 0; h < K9_V / 2; ++h)
            asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v[2 * h]), "=r"(v[2 * h + 1]) : "r"(at(stg, h)) : "memory");
    }
};

// store the lane's cells of an output row: 8-byte pieces on the fast path (the halo
// pairs at the strip ends are skipped), guarded scalar stores otherwise
__device__ __forceinline__ void k9_store(int32_t* row, bool vec, int lane, int xl,
                                         const int32_t (&out)[K9_V], const bool (&st)[K9_V],
                                         const Step2DArgs& a, unsigned& gacc)
{
    if (vec) {
#pragma unroll
        for (int h = 0; h < K9_V / 2; ++h) {
            const int p = lane * K9_V + 2 * h;
            if (p >= K9_H && p < K9_W - K9_H) {
                *reinterpret_cast<int2*>(row + xl + 2 * h) = make_int2(out[2 * h], out[2 * h + 1]);
                md_acc(gacc, out[2 * h], a.glo);
                md_acc(gacc, out[2 * h + 1], a.glo);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < K9_V; ++j)
            if (st[j]) {
                row[xl + j] = out[j];
                md_acc(gacc, out[j], a.glo);
            }
    }
}

template <int RULE, bool SAME>
struct GForm { static constexpr bool value = SAME && (RULE == R_EO_P1 || RULE == R_EO_FAST); };

template <int RULE, bool SAME>
struct Row2 {
    static constexpr bool G = GForm<RULE, SAME>::value;
    int32_t q[K9_V];
    int32_t g[G ? K9_V : 1], m[G ? K9_V : 1], pb[G ? K9_V : 1];
    int32_t px[G ? 1 : K9_V], mx[G ? 1 : K9_V], py[G ? 1 : K9_V], my[G ? 1 : K9_V];
    __device__ __forceinline__ void eval(const DevRule& rx, const DevRule& ry)
    {
#pragma unroll
        for (int j = 0; j < K9_V; ++j) {
            if constexpr (G) {
                if (j & 1) phi_gm<RULE, true, true>(q[j], g[j], m[j], rx);
                else phi_gm<RULE, false, true>(q[j], g[j], m[j], rx);
                pb[j] = g[j] - m[j];
            } else {
                phi_pm<RULE>(q[j], px[j], mx[j], rx);
                if (SAME) {
                    py[j] = px[j];
                    my[j] = mx[j];
                } else {
                    phi_pm<RULE>(q[j], py[j], my[j], ry);
                }
            }
        }
    }
};

// update of row C from rows B (below) and A (above); wall_* : transmissive ghost-copy
// transfers (the edge cell's own maps) at the domain boundary
template <int RULE, bool SAME, bool WALLS>
__device__ __forceinline__ void update_row(const Row2<RULE, SAME>& B, const Row2<RULE, SAME>& C,
                                           const Row2<RULE, SAME>& A, int xl, int nx, bool xwall,
                                           bool wall_lo, bool wall_hi, int32_t (&out)[K9_V])
{
    constexpr int V = K9_V;
    if constexpr (GForm<RULE, SAME>::value) {
        const int32_t pl = __shfl_up_sync(FULL2, C.pb[V - 1], 1);     // lane 0: halo, unused
        const int32_t mr = __shfl_down_sync(FULL2, C.m[0], 1);        // lane 31: halo, unused
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int32_t pbl = j > 0 ? C.pb[j - 1] : pl;
            const int32_t mrr = j + 1 < V ? C.m[j + 1] : mr;
            const int32_t w = 2 * C.m[j] - C.g[j];
            int32_t o = C.q[j] + pbl + B.pb[j] - mrr - A.m[j] + 2 * w;
            if (WALLS) {
                if (xwall) {
                    const int x = xl + j;
                    if (x == 0) o += C.pb[j] - pbl;                   // F_{-1/2} = phi+(q) + phi-(q)
                    if (x == nx - 1) o += mrr - C.m[j];
                }
                if (wall_lo) o += C.pb[j] - B.pb[j];
                if (wall_hi) o += A.m[j] - C.m[j];
            }
            out[j] = o;
        }
    } else {
        const int32_t pl = __shfl_up_sync(FULL2, C.px[V - 1], 1);
        const int32_t mr = __shfl_down_sync(FULL2, C.mx[0], 1);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            int32_t txl = (j > 0 ? C.px[j - 1] : pl) + C.mx[j];
            int32_t txr = C.px[j] + (j + 1 < V ? C.mx[j + 1] : mr);
            int32_t tyl = B.py[j] + C.my[j];
            int32_t tyr = C.py[j] + A.my[j];
            if (WALLS) {
                if (xwall) {
                    const int x = xl + j;
                    if (x == 0) txl = C.px[j] + C.mx[j];
                    if (x == nx - 1) txr = C.px[j] + C.mx[j];
                }
                if (wall_lo) tyl = C.py[j] + C.my[j];
                if (wall_hi) tyr = C.py[j] + C.my[j];
            }
            out[j] = C.q[j] + txl - txr + tyl - tyr;
        }
    }
}

template <int RULE, bool SAME>
__global__ void K9_LB1 k_step2d_s(Step2DArgs a, DevRule rx, DevRule ry)
{
    if (a.guard && *a.guard) return;                    // state left the range earlier
    unsigned gacc = 0;                                  // range guard: max (unsigned)(q - lo) seen
    constexpr int V = K9_V;
    const int lane = threadIdx.x & 31;
    const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nx = (int)a.nx, ny = (int)a.ny, bm = a.bmode;
    const int nstrips = (nx + K9_S - 1) / K9_S;
    const int yc = a.ksteps;                               // rows per chunk (launcher)
    const int nchunks = (ny + yc - 1) / yc;
    if (warp >= nstrips * nchunks) return;                 // whole warps only
    const int strip = warp % nstrips, chunk = warp / nstrips;
    const int x0 = strip * K9_S - K9_H;                     // first loaded column
    const int y0 = chunk * yc, y1 = (y0 + yc < ny) ? y0 + yc : ny;
    const int xl = x0 + lane * V;
    // int2 path: the strip lies inside the row and rows are 8-byte aligned
    const bool vec = x0 >= 0 && x0 + K9_W <= nx && (nx % 2 == 0);
    int xo[V];
#pragma unroll
    for (int j = 0; j < V; ++j) xo[j] = wrap2(xl + j, nx, bm);
    // stored cells of this lane: columns [x0 + H, x0 + W - H) inside [0, nx)
    bool st[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int p = lane * V + j, x = xl + j;
        st[j] = p >= K9_H && p < K9_W - K9_H && x >= 0 && x < nx;
    }

    // Row ring in shared memory: each lane streams its 4 cells K9_LOOK rows ahead with
    // cp.async (two 8-byte copies: strips start at x = 2 mod 4), one commit group per
    // row; a lane reads only the slots it filled, so no barrier is needed.
    // Stage of row r: (r - y0 + 1) % S.
    constexpr int L = K9_LOOK, S = K9_LOOK + 1;
    __shared__ int2 ring[S][256 / 32][K9_V / 2][32];
    K9Ring rg;
    rg.base = (unsigned)__cvta_generic_to_shared(&ring[0][threadIdx.x >> 5][0][lane]);
    auto issue = [&](int r, int stg) {
        if (r <= y1) rg.issue(stg, a.src + wrap_row(r, ny, bm) * nx, vec, xl, xo);   // rows beyond y1 are never read
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto read = [&](int stg, int32_t (&v)[V]) { rg.read(stg, v); };

    // one step: the clamped halo loads already are the transmissive ghost copies
    Row2<RULE, SAME> P0, P1, P2;
    for (int r = y0 - 1; r < y0 + L; ++r) issue(r, r - y0 + 1);   // rows y0 - 1 .. y0 + L - 1
    asm volatile("cp.async.wait_group %0;" :: "n"(L - 1) : "memory");   // rows y0 - 1, y0 landed
    read(0, P2.q);
    P2.eval(rx, ry);                                       // row y0 - 1
    read(1, P0.q);
    P0.eval(rx, ry);
    int sz = 1;                                            // stage of row r
    // one row: C = row r, Nn = row r + 1 (read from the ring, maps evaluated here),
    // Bp = row r - 1
    auto body = [&](int r, Row2<RULE, SAME>& Bp, Row2<RULE, SAME>& C, Row2<RULE, SAME>& Nn) {
        const int sn = sz + 1 == S ? 0 : sz + 1, sl = sz == 0 ? S - 1 : sz - 1;
        asm volatile("cp.async.wait_group %0;" :: "n"(L - 2) : "memory");  // rows <= r + 1
        read(sn, Nn.q);
        issue(r + L, sl);                                  // into row r - 1's stage
        Nn.eval(rx, ry);
        int32_t out[V];
        update_row<RULE, SAME, false>(Bp, C, Nn, xl, nx, false, false, false, out);
        k9_store(a.dst + r * nx, vec, lane, xl, out, st, a, gacc);
        sz = sn;
    };
    int r = y0;
    for (; r + 3 <= y1; r += 3) {
        body(r, P2, P0, P1);
        body(r + 1, P0, P1, P2);
        body(r + 2, P1, P2, P0);
    }
    if (r < y1) body(r, P2, P0, P1);
    if (r + 1 < y1) body(r + 1, P0, P1, P2);
    asm volatile("cp.async.wait_all;" ::: "memory");
    md_flush(a.guard, gacc, a.glo, a.ghi);
}

// K9 with two steps per launch (temporal blocking k = 2): the warp streams the step-0
// rows, computes step-1 row t-1 as soon as step-0 row t has arrived and step-2 row t-2
// as soon as step-1 row t-1 exists; only step-2 rows are stored, so one HBM round trip
// advances two steps (4 B per cell-update).  The two halo columns on each side are
// exactly the dependence of two steps; a chunk recomputes two step-1 rows beyond each
// end.  Transmissive walls: the boundary transfer of every step uses the edge cell's
// own maps (ghost copy, reading A12), as the clamped halo no longer carries it.
template <int RULE, bool SAME>
__global__ void K9_LB2 k_step2d_s2(Step2DArgs a, DevRule rx, DevRule ry)
{
    if (a.guard && *a.guard) return;                    // state left the range earlier
    unsigned gacc = 0;                                  // range guard: max (unsigned)(q - lo) seen
    constexpr int V = K9_V, L = K9_LOOK;
    const int lane = threadIdx.x & 31;
    const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nx = (int)a.nx, ny = (int)a.ny, bm = a.bmode;
    const int nstrips = (nx + K9_S - 1) / K9_S;
    const int yc = a.ksteps;                               // rows per chunk (launcher)
    const int nchunks = (ny + yc - 1) / yc;
    if (warp >= nstrips * nchunks) return;
    const int strip = warp % nstrips, chunk = warp / nstrips;
    const int x0 = strip * K9_S - K9_H;
    const int y0 = chunk * yc, y1 = (y0 + yc < ny) ? y0 + yc : ny;
    const int xl = x0 + lane * V;
    const bool vec = x0 >= 0 && x0 + K9_W <= nx && (nx % 2 == 0);
    const bool wall = bm == BM_TRANSMISSIVE;
    const bool xwall = wall && (x0 <= 0 || x0 + K9_W - 1 >= nx - 1);      // a wall is in the strip
    int xo[V];
#pragma unroll
    for (int j = 0; j < V; ++j) xo[j] = wrap2(xl + j, nx, bm);
    bool stc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int p = lane * V + j, x = xl + j;
        stc[j] = p >= K9_H && p < K9_W - K9_H && x >= 0 && x < nx;
    }
    bool ck1[V];                                           // valid step-1 cells of the strip
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int p = lane * V + j, x = xl + j;
        ck1[j] = p >= 1 && p < K9_W - 1 && x >= 0 && x < nx;
    }
    __shared__ int2 ring[L][256 / 32][K9_V / 2][32];
    K9Ring rg;
    rg.base = (unsigned)__cvta_generic_to_shared(&ring[0][threadIdx.x >> 5][0][lane]);
    const int t0 = y0 - 2, t1 = y1 + 1;                    // step-0 rows streamed
    auto issue = [&](int t, int stg) {
        if (t <= t1) rg.issue(stg, a.src + wrap_row(t, ny, bm) * nx, vec, xl, xo);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int i = 0; i < L; ++i) issue(t0 + i, i);
    // three rotating slots per stage (step-0 rows t-2, t-1, t; step-1 rows t-3, t-2,
    // t-1), the loop unrolled by three so the rotation needs no register moves
    Row2<RULE, SAME> P0, P1, P2, Q0, Q1, Q2;
    int stg = 0;
    auto body = [&](int t, Row2<RULE, SAME>& A0, Row2<RULE, SAME>& B0, Row2<RULE, SAME>& C0,
                    Row2<RULE, SAME>& A1, Row2<RULE, SAME>& B1, Row2<RULE, SAME>& C1) {
        asm volatile("cp.async.wait_group %0;" :: "n"(L - 1) : "memory");  // row t landed
        rg.read(stg, C0.q);
        issue(t + L, stg);                                 // the row just read is free
        stg = stg + 1 == L ? 0 : stg + 1;
        C0.eval(rx, ry);
        if (t >= y0) {                                     // step-1 row t - 1
            const int r = t - 1;
            if (wall) update_row<RULE, SAME, true>(A0, B0, C0, xl, nx, xwall, r == 0, r == ny - 1, C1.q);
            else update_row<RULE, SAME, false>(A0, B0, C0, xl, nx, false, false, false, C1.q);
            if (a.guard && r >= 0 && r < ny) {             // range guard on the step-1 row
#pragma unroll
                for (int j = 0; j < V; ++j)
                    if (ck1[j]) md_acc(gacc, C1.q[j], a.glo);
            }
            C1.eval(rx, ry);
            if (t >= y0 + 2) {                             // step-2 row t - 2: store
                const int r2 = t - 2;
                int32_t out[V];
                if (wall) update_row<RULE, SAME, true>(A1, B1, C1, xl, nx, xwall, r2 == 0, r2 == ny - 1, out);
                else update_row<RULE, SAME, false>(A1, B1, C1, xl, nx, false, false, false, out);
                k9_store(a.dst + r2 * nx, vec, lane, xl, out, stc, a, gacc);
            }
        }
    };
    const int niter = t1 - t0 + 1;
    int i = 0;
    for (; i + 3 <= niter; i += 3) {
        body(t0 + i, P1, P2, P0, Q0, Q1, Q2);
        body(t0 + i + 1, P2, P0, P1, Q1, Q2, Q0);
        body(t0 + i + 2, P0, P1, P2, Q2, Q0, Q1);
    }
    if (i < niter) body(t0 + i, P1, P2, P0, Q0, Q1, Q2);
    if (i + 1 < niter) body(t0 + i + 1, P2, P0, P1, Q1, Q2, Q0);
    asm volatile("cp.async.wait_all;" ::: "memory");
    md_flush(a.guard, gacc, a.glo, a.ghi);
}

template <int RULE>
static cudaError_t s2d2_rule(bool same, const Step2DArgs& a, const DevRule& rx, const DevRule& ry,
                             cudaStream_t st)
{
    const int64_t strips = (a.nx + K9_S - 1) / K9_S;
    const int64_t chunks = (a.ny + a.ksteps - 1) / a.ksteps;
    const unsigned grid = (unsigned)((strips * chunks * 32 + 255) / 256);
    if (same) k_step2d_s2<RULE, true><<<grid, 256, 0, st>>>(a, rx, ry);
    else k_step2d_s2<RULE, false><<<grid, 256, 0, st>>>(a, rx, ry);
    return cudaGetLastError();
}

// two time steps per launch (a.ksteps carries the rows per chunk)
cudaError_t launch_step2d_stream2(int rule, bool same, const Step2DArgs& a, const DevRule& rx,
                                  const DevRule& ry, cudaStream_t st)
{
    if (a.ksteps < 1) return cudaErrorInvalidValue;
    switch (rule) {
        case R_LIN_HALF: return s2d2_rule<R_LIN_HALF>(same, a, rx, ry, st);
        case R_EO_FAST: return s2d2_rule<R_EO_FAST>(same, a, rx, ry, st);
        case R_EO_P1: return s2d2_rule<R_EO_P1>(same, a, rx, ry, st);
        case R_GENERIC: return s2d2_rule<R_GENERIC>(same, a, rx, ry, st);
        case R_LIN_FAST: return s2d2_rule<R_LIN_FAST>(same, a, rx, ry, st);
        default: return cudaErrorInvalidValue;
    }
}

int64_t step2d_stream_rows(int64_t nx, int64_t ny)
{
    const int64_t strips = (nx + K9_S - 1) / K9_S;
#ifndef FQNM_K9_WARPS_PER_SM
#define FQNM_K9_WARPS_PER_SM 48
#endif
    int64_t yc = strips * ny / (148 * FQNM_K9_WARPS_PER_SM);   // ~48 warps per SM in total
    if (yc < 8) yc = 8;
    if (yc > 512) yc = 512;
    if (yc >= ny) return ny;
#ifndef FQNM_K9_RAGGED
    const int64_t nch = (ny + yc - 1) / yc;                // equal chunks, no short tail
    yc = (ny + nch - 1) / nch;
#endif
    return yc;
}

template <int RULE>
static cudaError_t s2d_rule(bool same, const Step2DArgs& a, const DevRule& rx, const DevRule& ry,
                            cudaStream_t st)
{
    const int64_t strips = (a.nx + K9_S - 1) / K9_S;
    const int64_t chunks = (a.ny + a.ksteps - 1) / a.ksteps;
    const int64_t threads = strips * chunks * 32;
    const unsigned grid = (unsigned)((threads + 255) / 256);
    if (same) k_step2d_s<RULE, true><<<grid, 256, 0, st>>>(a, rx, ry);
    else k_step2d_s<RULE, false><<<grid, 256, 0, st>>>(a, rx, ry);
    return cudaGetLastError();
}

// a.ksteps carries the rows per chunk (step2d_stream_rows); one time step per launch
cudaError_t launch_step2d_stream(int rule, bool same, const Step2DArgs& a, const DevRule& rx,
                                 const DevRule& ry, cudaStream_t st)
{
    if (a.ksteps < 1) return cudaErrorInvalidValue;
    switch (rule) {
        case R_LIN_HALF: return s2d_rule<R_LIN_HALF>(same, a, rx, ry, st);
        case R_EO_FAST: return s2d_rule<R_EO_FAST>(same, a, rx, ry, st);
        case R_EO_P1: return s2d_rule<R_EO_P1>(same, a, rx, ry, st);
        case R_GENERIC: return s2d_rule<R_GENERIC>(same, a, rx, ry, st);
        case R_LIN_FAST: return s2d_rule<R_LIN_FAST>(same, a, rx, ry, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fqnm
