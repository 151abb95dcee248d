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
static constexpr int K9_V = 4;                  // x cells per lane
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

template <int RULE, bool SAME>
struct Maps2 {
    int32_t px[K9_V], mx[K9_V], py[K9_V], my[K9_V];
    __device__ __forceinline__ void eval(const int32_t (&q)[K9_V], const DevRule& rx,
                                         const DevRule& ry)
    {
#pragma unroll
        for (int j = 0; j < K9_V; ++j) {
            phi_pm<RULE>(q[j], px[j], mx[j], rx);
            if (SAME) {
                py[j] = px[j];
                my[j] = mx[j];
            } else {
                phi_pm<RULE>(q[j], py[j], my[j], ry);
            }
        }
    }
};

template <int RULE, bool SAME>
__global__ void __launch_bounds__(256) k_step2d_s(Step2DArgs a, DevRule rx, DevRule ry)
{
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
    __shared__ int4 ring[S][256 / 32][32];
    const int wib = threadIdx.x >> 5;
    const unsigned ring0 = (unsigned)__cvta_generic_to_shared(&ring[0][wib][lane]);
    constexpr unsigned RSTRIDE = sizeof(ring[0]);
    auto issue = [&](int r, int stg) {
        if (r <= y1) {                                     // rows beyond y1 are never read
            const int32_t* row = a.src + wrap_row(r, ny, bm) * nx;
            const unsigned d = ring0 + stg * RSTRIDE;
            if (vec) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(row + xl) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d + 8), "l"(row + xl + 2) : "memory");
            } else {
#pragma unroll
                for (int j = 0; j < V; ++j)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d + 4 * j), "l"(row + xo[j]) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto read = [&](int stg, int32_t (&v)[V]) {
        int4 t;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "r"(ring0 + stg * RSTRIDE) : "memory");
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    };

    Maps2<RULE, SAME> M0, M1, M2;
    int32_t Q0[V], Q1[V], Q2[V];
    for (int r = y0 - 1; r < y0 + L; ++r) issue(r, r - y0 + 1);   // rows y0 - 1 .. y0 + L - 1
    asm volatile("cp.async.wait_group %0;" :: "n"(L - 1) : "memory");   // rows y0 - 1, y0 landed
    read(0, Q2);
    M2.eval(Q2, rx, ry);                                   // row y0 - 1 (its phi+_y)
    read(1, Q0);
    M0.eval(Q0, rx, ry);
    int sz = 1;                                            // stage of row r
    // one row: Qc/Mc = row r, Qn/Mn = row r + 1 (read from the ring, maps evaluated
    // here), Mp = row r - 1
    auto body = [&](int r, int32_t (&Qc)[V], int32_t (&Qn)[V], Maps2<RULE, SAME>& Mp,
                    Maps2<RULE, SAME>& Mc, Maps2<RULE, SAME>& Mn) {
        const int sn = sz + 1 == S ? 0 : sz + 1, sl = sz == 0 ? S - 1 : sz - 1;
        asm volatile("cp.async.wait_group %0;" :: "n"(L - 2) : "memory");  // rows <= r + 1
        read(sn, Qn);
        issue(r + L, sl);                                  // into row r - 1's stage
        Mn.eval(Qn, rx, ry);
        const int32_t pl = __shfl_up_sync(FULL2, Mc.px[V - 1], 1);   // lane 0: halo cell, unused
        const int32_t mr = __shfl_down_sync(FULL2, Mc.mx[0], 1);     // lane 31: halo, unused
        // transmissive walls need no special case: the clamped halo loads make the
        // wall transfer phi+(q_e) + phi-(q_e) (ghost copy, reading A12)
        int32_t out[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int32_t txl = (j > 0 ? Mc.px[j - 1] : pl) + Mc.mx[j];        // F^x_{i-1/2}
            const int32_t txr = Mc.px[j] + (j + 1 < V ? Mc.mx[j + 1] : mr);    // F^x_{i+1/2}
            const int32_t tyl = Mp.py[j] + Mc.my[j];                           // F^y_{j-1/2}
            const int32_t tyr = Mc.py[j] + Mn.my[j];                           // F^y_{j+1/2}
            out[j] = Qc[j] + txl - txr + tyl - tyr;
        }
        // (transmissive rows: wrap_row clamps, so the ghost rows repeat the edge row)
        int32_t* row = a.dst + r * nx;
        if (vec) {
            if (lane > 0 && lane < 31) {
                *reinterpret_cast<int2*>(row + xl) = make_int2(out[0], out[1]);
                *reinterpret_cast<int2*>(row + xl + 2) = make_int2(out[2], out[3]);
            } else if (lane == 0) {
                *reinterpret_cast<int2*>(row + xl + 2) = make_int2(out[2], out[3]);
            } else {
                *reinterpret_cast<int2*>(row + xl) = make_int2(out[0], out[1]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (st[j]) row[xl + j] = out[j];
        }
        sz = sn;
    };
    int r = y0;
    for (; r + 3 <= y1; r += 3) {
        body(r, Q0, Q1, M2, M0, M1);
        body(r + 1, Q1, Q2, M0, M1, M2);
        body(r + 2, Q2, Q0, M1, M2, M0);
    }
    if (r < y1) body(r, Q0, Q1, M2, M0, M1);
    if (r + 1 < y1) body(r + 1, Q1, Q2, M0, M1, M2);
    asm volatile("cp.async.wait_all;" ::: "memory");
}

int64_t step2d_stream_rows(int64_t nx, int64_t ny)
{
    const int64_t strips = (nx + K9_S - 1) / K9_S;
    int64_t yc = strips * ny / (148 * 48);                 // ~48 warps per SM in total
    if (yc < 8) yc = 8;
    if (yc > 512) yc = 512;
    return yc < ny ? yc : ny;
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
