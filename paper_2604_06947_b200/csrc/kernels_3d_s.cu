// K10: 3D directional composition, warp streaming (Thm formal Cartesian dimensional
// extension, Eq. nd_transfer_rule with d = 3):
//   q'_c = q_c - sum_{m = x,y,z} (F_{c+1/2 e_m} - F_{c-1/2 e_m}),
//   F_{c+1/2 e_m} = phi+_m(q_c) + phi-_m(q_{c+e_m}).
// One step per launch; no shared-memory exchange between warps and no barriers.
// A warp owns two consecutive rows (y, y+1) of a 124-wide x strip and marches them
// through a chunk of z planes.  It loads four rows per plane (y-1 .. y+2; the outer two
// are y halo) of 128 columns (4 per lane, the outer 2 columns on each side are x halo),
// so every y neighbour's map is computed by the warp itself (2 maps per owned cell)
// and x neighbours come from registers and shuffles.  z neighbours' maps stay in
// registers: the owned rows' maps are evaluated one plane ahead.  The four rows of a
// plane stream through a per-warp shared-memory ring, K10_LOOK planes in flight per
// lane (cp.async, a lane reads only the slots it filled).
// HBM: 8 B per cell-update (the halo rows and columns are re-read from L2).
// Indices are 32-bit (nx * ny * nz < 2^31).
#include <cstdint>
#include <cuda_runtime.h>

#include "fqnm_internal.h"
#include "maps.cuh"

namespace fqnm {

static constexpr unsigned FULLS = 0xffffffffu;
static constexpr int K10_V = 4;                 // x cells per lane
static constexpr int K10_W = 32 * K10_V;        // loaded strip width
static constexpr int K10_H = 2;                 // x halo columns per side
static constexpr int K10_S = K10_W - 2 * K10_H; // strip stride
static constexpr int K10_R = 2;                 // owned rows per warp
static constexpr int K10_LOOK = 4;              // planes in flight per lane
static constexpr int K10_WARPS = 4;             // warps per CTA

__device__ __forceinline__ int wrap_s(int i, int n, int bmode)
{
    if (bmode == BM_PERIODIC) { i %= n; return i < 0 ? i + n : i; }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);            // transmissive ghost copy
}

__device__ __forceinline__ int wrap_near_s(int i, int n, int bmode)
{
    if (bmode == BM_PERIODIC) {
        if (i < 0) i += n;
        if (i < 0) i += n;
        if (i >= n) i -= n;
        if (i >= n) i -= n;
        return i;
    }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// maps of the owned rows' cells (R rows x V cells) in the three directions
template <int RULE, bool SAME>
struct OwnMaps {
    int32_t px[K10_R][K10_V], mx[K10_R][K10_V], py[K10_R][K10_V], my[K10_R][K10_V];
    int32_t pz[K10_R][K10_V], mz[K10_R][K10_V];
    __device__ __forceinline__ void eval(const int32_t (&q)[K10_R][K10_V], const DevRule& rx,
                                         const DevRule& ry, const DevRule& rz)
    {
#pragma unroll
        for (int i = 0; i < K10_R; ++i)
#pragma unroll
            for (int j = 0; j < K10_V; ++j) {
                phi_pm<RULE>(q[i][j], px[i][j], mx[i][j], rx);
                if (SAME) {
                    py[i][j] = pz[i][j] = px[i][j];
                    my[i][j] = mz[i][j] = mx[i][j];
                } else {
                    phi_pm<RULE>(q[i][j], py[i][j], my[i][j], ry);
                    phi_pm<RULE>(q[i][j], pz[i][j], mz[i][j], rz);
                }
            }
    }
};

template <int RULE, bool SAME>
__global__ void __launch_bounds__(32 * K10_WARPS) k_step3d_s(Step3DArgs a, DevRule rx, DevRule ry,
                                                           DevRule rz)
{
    if (a.guard && *a.guard) return;                    // state left the range earlier
    unsigned gacc = 0;                                  // range guard accumulator (md_acc)
    constexpr int V = K10_V, R = K10_R, L = K10_LOOK, S = K10_LOOK + 1;
    constexpr int NR = R + 2;                              // loaded rows per plane
    __shared__ int4 ring[S][K10_WARPS][NR][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int warp = blockIdx.x * K10_WARPS + wib;
    const int nx = (int)a.nx, ny = (int)a.ny, nz = (int)a.nz, bm = a.bmode;
    const int plane = nx * ny;
    const int nstrips = (nx + K10_S - 1) / K10_S;
    const int npairs = (ny + R - 1) / R;
    const int zc = (int)a.zchunk;
    const int nchunks = (nz + zc - 1) / zc;
    if (warp >= nstrips * npairs * nchunks) return;       // whole warps only
    const int strip = warp % nstrips;
    const int pair = (warp / nstrips) % npairs;
    const int chunk = warp / (nstrips * npairs);
    const int x0 = strip * K10_S - K10_H, y0 = pair * R;
    const int z0 = chunk * zc, z1 = (z0 + zc < nz) ? z0 + zc : nz;
    const int xl = x0 + lane * V;
    const bool vec = x0 >= 0 && x0 + K10_W <= nx && (nx % 2 == 0);
    int xo[V];
#pragma unroll
    for (int j = 0; j < V; ++j) xo[j] = wrap_s(xl + j, nx, bm);
    int rowoff[NR];                                        // rows y0-1 .. y0+R
#pragma unroll
    for (int i = 0; i < NR; ++i) rowoff[i] = wrap_s(y0 - 1 + i, ny, bm) * nx;
    bool stc[V];                                           // stored columns of the lane
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int pcol = lane * V + j, x = xl + j;
        stc[j] = pcol >= K10_H && pcol < K10_W - K10_H && x >= 0 && x < nx;
    }
    const unsigned ring0 = (unsigned)__cvta_generic_to_shared(&ring[0][wib][0][lane]);
    constexpr unsigned SSTRIDE = sizeof(ring[0]), RSTRIDE = sizeof(ring[0][0][0]);

    // stage of plane p: (p - z0 + 1) % S
    auto issue = [&](int p, int stg) {
        if (p <= z1) {                                     // planes beyond z1 are never read
            const int32_t* pl = a.src + wrap_near_s(p, nz, bm) * plane;
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const unsigned d = ring0 + stg * SSTRIDE + i * RSTRIDE;
                const int32_t* row = pl + rowoff[i];
                if (vec) {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(row + xl) : "memory");
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d + 8), "l"(row + xl + 2) : "memory");
                } else {
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d + 4 * j), "l"(row + xo[j]) : "memory");
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto read_row = [&](int stg, int i, int32_t (&v)[V]) {
        int4 t;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                     : "r"(ring0 + stg * SSTRIDE + i * RSTRIDE) : "memory");
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    };
    auto read_own = [&](int stg, int32_t (&q)[R][V]) {
#pragma unroll
        for (int i = 0; i < R; ++i) read_row(stg, i + 1, q[i]);
    };

    OwnMaps<RULE, SAME> MA, MB;
    int32_t pzb[R][V];
    for (int p = z0 - 1; p < z0 + L; ++p) issue(p, p - z0 + 1);
    asm volatile("cp.async.wait_group %0;" :: "n"(L - 1) : "memory");   // planes z0 - 1, z0
    {
        int32_t q[R][V];
        read_own(0, q);
        MB.eval(q, rx, ry, rz);                            // plane z0 - 1: its phi+_z
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int j = 0; j < V; ++j) pzb[i][j] = MB.pz[i][j];
        read_own(1, q);
        MA.eval(q, rx, ry, rz);
    }
    int sz = 1;
    // one plane: Mc = maps of plane z (owned rows), Mn = plane z + 1 (evaluated here)
    auto body = [&](int z, OwnMaps<RULE, SAME>& Mc, OwnMaps<RULE, SAME>& Mn) {
        const int sn = sz + 1 == S ? 0 : sz + 1, sl = sz == 0 ? S - 1 : sz - 1;
        asm volatile("cp.async.wait_group %0;" :: "n"(L - 2) : "memory");  // planes <= z + 1
        {
            int32_t q[R][V];
            read_own(sn, q);
            Mn.eval(q, rx, ry, rz);                        // plane z + 1
        }
        // y halo rows of plane z: phi+_y of row y0 - 1, phi-_y of row y0 + R
        int32_t pyd[V], myu[V];
        {
            int32_t h0[V], h1[V];
            read_row(sz, 0, h0);
            read_row(sz, NR - 1, h1);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                int32_t p_, m_;
                phi_pm<RULE>(h0[j], pyd[j], m_, ry);
                phi_pm<RULE>(h1[j], p_, myu[j], ry);
            }
        }
        int32_t qc[R][V];
        read_own(sz, qc);
        issue(z + L, sl);                                  // into plane z - 1's stage
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int32_t pl = __shfl_up_sync(FULLS, Mc.px[i][V - 1], 1);    // lane 0: halo
            const int32_t mr = __shfl_down_sync(FULLS, Mc.mx[i][0], 1);      // lane 31: halo
            const int y = y0 + i;
            int32_t out[V];
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int32_t pxl = j > 0 ? Mc.px[i][j - 1] : pl;
                const int32_t mxr = j + 1 < V ? Mc.mx[i][j + 1] : mr;
                const int32_t pyl = i > 0 ? Mc.py[i - 1][j] : pyd[j];
                const int32_t myr = i + 1 < R ? Mc.my[i + 1][j] : myu[j];
                const int32_t dF = (Mc.px[i][j] + mxr) - (pxl + Mc.mx[i][j]) +
                                   (Mc.py[i][j] + myr) - (pyl + Mc.my[i][j]) +
                                   (Mc.pz[i][j] + Mn.mz[i][j]) - (pzb[i][j] + Mc.mz[i][j]);
                out[j] = qc[i][j] - dF;
            }
            if (y < ny) {
                int32_t* row = a.dst + z * plane + y * nx;
                if (vec) {
                    if (lane > 0 && lane < 31) {
                        *reinterpret_cast<int2*>(row + xl) = make_int2(out[0], out[1]);
                        *reinterpret_cast<int2*>(row + xl + 2) = make_int2(out[2], out[3]);
                    } else if (lane == 0) {
                        *reinterpret_cast<int2*>(row + xl + 2) = make_int2(out[2], out[3]);
                    } else {
                        *reinterpret_cast<int2*>(row + xl) = make_int2(out[0], out[1]);
                    }
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if ((lane > 0 || j >= 2) && (lane < 31 || j < 2)) md_acc(gacc, out[j], a.glo);
                } else {
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (stc[j]) {
                            row[xl + j] = out[j];
                            md_acc(gacc, out[j], a.glo);
                        }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int j = 0; j < V; ++j) pzb[i][j] = Mc.pz[i][j];
        sz = sn;
    };
    int z = z0;
    for (; z + 2 <= z1; z += 2) {
        body(z, MA, MB);
        body(z + 1, MB, MA);
    }
    if (z < z1) body(z, MA, MB);
    asm volatile("cp.async.wait_all;" ::: "memory");
    md_flush(a.guard, gacc, a.glo, a.ghi);
}

int64_t step3d_s_zchunk(int64_t nx, int64_t ny, int64_t nz)
{
    const int64_t cols = ((nx + K10_S - 1) / K10_S) * ((ny + K10_R - 1) / K10_R);
    int64_t zc = cols * nz / (148 * 64);                   // ~64 warps per SM in total
    if (zc < 8) zc = 8;
    if (zc > 256) zc = 256;
    return zc < nz ? zc : nz;
}

template <int RULE>
static cudaError_t s3d_rule(bool same, const Step3DArgs& a, const DevRule& rx, const DevRule& ry,
                            const DevRule& rz, cudaStream_t st)
{
    const int64_t warps = ((a.nx + K10_S - 1) / K10_S) * ((a.ny + K10_R - 1) / K10_R) *
                          ((a.nz + a.zchunk - 1) / a.zchunk);
    const unsigned grid = (unsigned)((warps + K10_WARPS - 1) / K10_WARPS);
    if (same) k_step3d_s<RULE, true><<<grid, 32 * K10_WARPS, 0, st>>>(a, rx, ry, rz);
    else k_step3d_s<RULE, false><<<grid, 32 * K10_WARPS, 0, st>>>(a, rx, ry, rz);
    return cudaGetLastError();
}

cudaError_t launch_step3d_stream(int rule, bool same, const Step3DArgs& a, const DevRule& rx,
                                 const DevRule& ry, const DevRule& rz, cudaStream_t st)
{
    if (a.zchunk < 1) return cudaErrorInvalidValue;
    switch (rule) {
        case R_LIN_HALF: return s3d_rule<R_LIN_HALF>(same, a, rx, ry, rz, st);
        case R_EO_FAST: return s3d_rule<R_EO_FAST>(same, a, rx, ry, rz, st);
        case R_EO_P1: return s3d_rule<R_EO_P1>(same, a, rx, ry, rz, st);
        case R_GENERIC: return s3d_rule<R_GENERIC>(same, a, rx, ry, rz, st);
        case R_LIN_FAST: return s3d_rule<R_LIN_FAST>(same, a, rx, ry, rz, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fqnm
