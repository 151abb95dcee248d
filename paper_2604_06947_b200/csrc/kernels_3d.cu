// K8: 3D directional composition (Thm formal Cartesian dimensional extension,
// PAPER.md P:364-401, Eq. nd_transfer_rule with d = 3):
//   q'_c = q_c - sum_{m = x,y,z} (F_{c+1/2 e_m} - F_{c-1/2 e_m}),
//   F_{c+1/2 e_m} = phi+_m(q_c) + phi-_m(q_{c+e_m}).
// One step per launch, 2.5D streaming through z.  A CTA of 10 warps owns a
// 128 x 8 (x, y) tile and marches it through a chunk of z planes:
//   * warp w handles row y0 + w - 1; warps 1..8 own the tile's rows, warps 0 and 9
//     are the y halo rows (maps only, 25% extra map work);
//   * a lane holds 4 consecutive x cells (int4 loads/stores); x neighbours come
//     from the lane's own registers and warp shuffles, the two cells beyond the
//     tile's x edges are evaluated by lanes 0 and 31;
//   * y neighbours' maps are exchanged through shared memory (one row per warp),
//     z neighbours' maps stay in registers: every own cell's maps are evaluated
//     once, one plane ahead;
//   * the state streams through a shared-memory ring, K8_LOOK planes in flight per
//     thread (cp.async), enough bytes in flight to cover HBM latency.
// HBM traffic: the state is read and written once per step, 8 B per cell-update
// (int32), plus the halo rows (L2 hits for interior tiles).
// Indices are 32-bit (the planner guarantees nx * ny * nz < 2^31).
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "fqnm_internal.h"
#include "maps.cuh"

namespace fqnm {

static constexpr unsigned FULL3 = 0xffffffffu;
static constexpr int K8_V = 4;                  // x cells per lane
static constexpr int K8_TX = 32 * K8_V;         // tile width (x)
#ifndef FQNM_K8_TY
#define FQNM_K8_TY 8
#endif
static constexpr int K8_TY = FQNM_K8_TY;        // owned rows (y)
static constexpr int K8_WARPS = K8_TY + 2;      // + 2 halo rows
#ifndef FQNM_K8_LOOK
#define FQNM_K8_LOOK 6
#endif
static constexpr int K8_LOOK = FQNM_K8_LOOK;    // planes in flight per thread (cp.async ring)
// resident CTAs per SM asked of ptxas: 2 for the EO rules (98 -> 88 registers, so two
// 320-thread CTAs fit the register file: 459 vs 357 GCUPS at 512^3); the other rules fit
// two CTAs uncapped and run slower capped (linear 449 vs 391; profiles/r01_3d.jsonl)
#ifndef FQNM_K8_MINB
#define FQNM_K8_MINB 0
#endif
template <int RULE>
constexpr int k8_minb() { return FQNM_K8_MINB ? FQNM_K8_MINB : ((RULE == R_EO_P1 || RULE == R_EO_FAST) ? 2 : 1); }

__device__ __forceinline__ int wrap_i(int i, int n, int bmode)
{
    if (bmode == BM_PERIODIC) { i %= n; return i < 0 ? i + n : i; }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);            // transmissive ghost copy
}

// plane index z in [-2n, 2n) without a division
__device__ __forceinline__ int wrap_z(int z, int n, int bmode)
{
    if (bmode == BM_PERIODIC) {
        if (z < 0) z += n;
        if (z < 0) z += n;
        if (z >= n) z -= n;
        if (z >= n) z -= n;
        return z;
    }
    return z < 0 ? 0 : (z >= n ? n - 1 : z);
}

// maps of one cell for the three directions (SAME: one evaluation serves all)
// G form (one EO rule for all directions): g = phi+ + phi- kept with the constant
// bias of maps.cuh eo_gm_p1, m = phi-, p* = g - m (phi+ plus the bias); the update
//   q' = q + p_xl + p_yd + p_zd - m_xr - m_yu - m_zu + 3 (2 m_c - g_c)
// is free of the bias (+3 from the three p terms, -3 from the last term).
template <int RULE, bool SAME>
struct GForm3 { static constexpr bool value = SAME && (RULE == R_EO_P1 || RULE == R_EO_FAST); };

template <int RULE, bool SAME>
struct Maps3 {
    int32_t px, mx, py, my, pz, mz, g;
    __device__ __forceinline__ void eval(int32_t q, const DevRule& rx, const DevRule& ry,
                                         const DevRule& rz)
    {
        if constexpr (GForm3<RULE, SAME>::value) {
            phi_gm<RULE, false, true>(q, g, mx, rx);
            px = g - mx;
            py = pz = px;
            my = mz = mx;
        } else {
            phi_pm<RULE>(q, px, mx, rx);
            if (SAME) {
                py = pz = px;
                my = mz = mx;
            } else {
                phi_pm<RULE>(q, py, my, ry);
                phi_pm<RULE>(q, pz, mz, rz);
            }
        }
    }
};

// VEC: every tile of the launch is a full 128-cell row segment with nx % 4 == 0 (int4
// loads/stores); otherwise scalar accesses with wrapped x offsets (the last partial
// tile column, launched separately)
template <int RULE, bool SAME, bool VEC>
__global__ void __launch_bounds__(32 * K8_WARPS, k8_minb<RULE>()) k_step3d(Step3DArgs a, DevRule rx, DevRule ry,
                                                        DevRule rz)
{
    if (a.guard && *a.guard) return;                    // state left the range earlier
    unsigned gacc = 0;                                  // range guard: max (unsigned)(q - lo) seen
    constexpr int V = K8_V;
    // y maps of the plane, per row; double-buffered by plane parity so one barrier per
    // plane suffices (a warp writing buffer b for plane z + 2 has passed the barrier of
    // plane z + 1, which every warp reaches only after its reads of plane z)
    __shared__ int4 sPy[2][K8_WARPS][32], sMy[2][K8_WARPS][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nx = (int)a.nx, ny = (int)a.ny, nz = (int)a.nz, bm = a.bmode;
    const int plane = nx * ny;
    const int x0 = (blockIdx.x + a.xt0) * K8_TX, y0 = blockIdx.y * K8_TY;
    const int z0 = blockIdx.z * (int)a.zchunk;
    const int z1 = z0 + (int)a.zchunk < nz ? z0 + (int)a.zchunk : nz;
    const bool halo_row = (w == 0 || w == K8_WARPS - 1);     // warp-uniform
    const int yo = y0 + w - 1;                                // this warp's row
    const bool row_own = !halo_row && yo < ny;
    const int row = wrap_i(yo, ny, bm) * nx;                  // row offset inside a plane
    // x offsets of the lane's cells (wrapped / clamped beyond nx: they serve as
    // neighbours and never store)
    const int xl = x0 + lane * V;
    int xo[V];
#pragma unroll
    for (int j = 0; j < V; ++j) xo[j] = (xl + j < nx) ? xl + j : wrap_i(xl + j, nx, bm);
    constexpr bool vec = VEC;
    // the cell beyond the tile's x edge: lane 0 -> x0 - 1, lane 31 -> x0 + 128
    const bool edge_lane = (lane == 0 || lane == 31);
    const int xe = lane == 0 ? wrap_i(x0 - 1, nx, bm) : wrap_i(x0 + K8_TX, nx, bm);

    // Plane ring in shared memory: every thread streams its own 4 cells (and lanes
    // 0/31 of owned rows the x-edge cell) K8_LOOK planes ahead with cp.async, one
    // commit group per plane; a thread only ever reads the slots it filled, so the
    // ring needs no barrier of its own.  Stage of plane p: (p - z0 + 1) % S.
    constexpr int L = K8_LOOK, S = K8_LOOK + 1;
    // the ring lives in dynamic shared memory (static shared memory is capped at 48 KB)
    extern __shared__ int4 k8_dyn[];
    int4 (*ring)[K8_WARPS][32] = reinterpret_cast<int4 (*)[K8_WARPS][32]>(k8_dyn);
    __shared__ int32_t ering[S][K8_WARPS][2];
    const int eslot = lane == 0 ? 0 : 1;
    // shared-memory addresses of this thread's ring slots, computed once
    const unsigned ring0 = (unsigned)__cvta_generic_to_shared(&ring[0][w][lane]);
    const unsigned ering0 = (unsigned)__cvta_generic_to_shared(&ering[0][w][eslot]);
    constexpr unsigned RSTRIDE = K8_WARPS * 32 * sizeof(int4), ESTRIDE = sizeof(ering[0]);
    const int32_t* gsrc = a.src + row;
    auto issue = [&](int p, int st) {
        if (p <= z1) {                                     // planes beyond z1 are never read
            const int32_t* g = gsrc + wrap_z(p, nz, bm) * plane;
            const unsigned d = ring0 + st * RSTRIDE;
            if (vec) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(g + xl) : "memory");
            } else {
#pragma unroll
                for (int j = 0; j < V; ++j)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d + 4 * j), "l"(g + xo[j]) : "memory");
            }
            if (edge_lane && !halo_row)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(ering0 + st * ESTRIDE), "l"(g + xe) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto read = [&](int st, int32_t (&v)[V]) {
        int4 t;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "r"(ring0 + st * RSTRIDE) : "memory");
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    };
    auto read_edge = [&](int st) -> int32_t {
        int32_t e;
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(e) : "r"(ering0 + st * ESTRIDE) : "memory");
        return e;
    };
    auto next = [&](int st) { return st + 1 == S ? 0 : st + 1; };

    // Three rotating register sets (planes z - 1, z, z + 1 of the maps; z, z + 1 of the
    // state), the loop unrolled by three so the rotation needs no register moves.
    Maps3<RULE, SAME> M0[V], M1[V], M2[V];
    int32_t Q0[V], Q1[V], Q2[V];
    for (int p = z0 - 1; p < z0 + L; ++p) issue(p, p - z0 + 1);   // planes z0 - 1 .. z0 + L - 1
    if (!halo_row) {
        asm volatile("cp.async.wait_group %0;" :: "n"(L - 1) : "memory");   // z0 - 1, z0 landed
        read(0, Q2);
#pragma unroll
        for (int j = 0; j < V; ++j) M2[j].eval(Q2[j], rx, ry, rz);      // plane z0 - 1
        read(1, Q0);
#pragma unroll
        for (int j = 0; j < V; ++j) M0[j].eval(Q0[j], rx, ry, rz);
    }
    // one plane: Qc/Mc = plane z, Qn/Mn = plane z + 1 (own rows read it from the ring
    // and evaluate its maps here), Mp = plane z - 1 (its phi+_z)
    // stage indices: sz = stage of plane z, sn = of z + 1, sl = of z - 1 (= of z + L)
    int sz = 1, yb = 0;
    auto body = [&](int z, int32_t (&Qc)[V], int32_t (&Qn)[V], Maps3<RULE, SAME> (&Mp)[V],
                    Maps3<RULE, SAME> (&Mc)[V], Maps3<RULE, SAME> (&Mn)[V]) {
        const int sn = next(sz), sl = sz == 0 ? S - 1 : sz - 1;
        // issued so far: planes z0 - 1 .. z + L - 1; planes <= z + 1 must have landed
        asm volatile("cp.async.wait_group %0;" :: "n"(L - 2) : "memory");
        int32_t pl = 0, mr = 0;
        if (halo_row) {
            read(sz, Qc);
#pragma unroll
            for (int j = 0; j < V; ++j) Mc[j].eval(Qc[j], rx, ry, rz);
        } else {
            read(sn, Qn);
#pragma unroll
            for (int j = 0; j < V; ++j) Mn[j].eval(Qn[j], rx, ry, rz);   // plane z + 1
            Maps3<RULE, SAME> me;
            me.eval(read_edge(sz), rx, ry, rz);                // x-edge cell of plane z
            // x neighbours across lanes: phi+ left of cell 0, phi- right of cell V-1
            pl = __shfl_up_sync(FULL3, Mc[V - 1].px, 1);
            mr = __shfl_down_sync(FULL3, Mc[0].mx, 1);
            if (lane == 0) pl = me.px;
            if (lane == 31) mr = me.mx;
        }
        issue(z + L, sl);                                  // into plane z - 1's stage
        sPy[yb][w][lane] = make_int4(Mc[0].py, Mc[1].py, Mc[2].py, Mc[3].py);
        sMy[yb][w][lane] = make_int4(Mc[0].my, Mc[1].my, Mc[2].my, Mc[3].my);
        __syncthreads();
        if (!halo_row) {
            const int4 pd = sPy[yb][w - 1][lane];              // row below: phi+_y
            const int4 mu = sMy[yb][w + 1][lane];              // row above: phi-_y
            const int32_t pyd[V] = {pd.x, pd.y, pd.z, pd.w};
            const int32_t myu[V] = {mu.x, mu.y, mu.z, mu.w};
            int32_t out[V];
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int32_t pxl = j > 0 ? Mc[j - 1].px : pl;
                const int32_t mxr = j + 1 < V ? Mc[j + 1].mx : mr;
                if constexpr (GForm3<RULE, SAME>::value) {
                    out[j] = Qc[j] + pxl + pyd[j] + Mp[j].pz - mxr - myu[j] - Mn[j].mz +
                             3 * (2 * Mc[j].mx - Mc[j].g);
                } else {
                    const int32_t dF = (Mc[j].px + mxr) - (pxl + Mc[j].mx) +
                                       (Mc[j].py + myu[j]) - (pyd[j] + Mc[j].my) +
                                       (Mc[j].pz + Mn[j].mz) - (Mp[j].pz + Mc[j].mz);
                    out[j] = Qc[j] - dF;
                }
            }
            if (row_own) {
                const int base = z * plane + row;
                if (vec) {
                    *reinterpret_cast<int4*>(a.dst + base + xl) =
                        make_int4(out[0], out[1], out[2], out[3]);
#pragma unroll
                    for (int j = 0; j < V; ++j) md_acc(gacc, out[j], a.glo);
                } else {
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (xl + j < nx) {
                            a.dst[base + xl + j] = out[j];
                            md_acc(gacc, out[j], a.glo);
                        }
                }
            }
        }
        yb ^= 1;
        sz = sn;
    };
    int z = z0;
    for (; z + 3 <= z1; z += 3) {
        body(z, Q0, Q1, M2, M0, M1);
        body(z + 1, Q1, Q2, M0, M1, M2);
        body(z + 2, Q2, Q0, M1, M2, M0);
    }
    if (z < z1) body(z, Q0, Q1, M2, M0, M1);
    if (z + 1 < z1) body(z + 1, Q1, Q2, M0, M1, M2);
    asm volatile("cp.async.wait_all;" ::: "memory");
    md_flush(a.guard, gacc, a.glo, a.ghi);
}

template <int RULE>
static cudaError_t step3d_rule(bool same, const Step3DArgs& a0, const DevRule& rx,
                               const DevRule& ry, const DevRule& rz, cudaStream_t st)
{
    Step3DArgs a = a0;
    dim3 block(32 * K8_WARPS);
    constexpr size_t dyn = (size_t)(K8_LOOK + 1) * K8_WARPS * 32 * sizeof(int4);
    // once per instantiation and device (devices >= 64: every launch); atomic, so host
    // threads launching concurrently do not race on the mask
    static std::atomic<unsigned long long> attr_set{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64 || !(attr_set.load() >> dev & 1ull)) {
        for (auto f : {k_step3d<RULE, true, true>, k_step3d<RULE, false, true>,
                       k_step3d<RULE, true, false>, k_step3d<RULE, false, false>}) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)dyn);
            if (e != cudaSuccess) return e;
        }
        if (dev < 64) attr_set.fetch_or(1ull << dev);
    }
    const unsigned gy = (unsigned)((a.ny + K8_TY - 1) / K8_TY);
    const unsigned gz = (unsigned)((a.nz + a.zchunk - 1) / a.zchunk);
    // full 128-wide tiles on the int4 path, the partial last tile column separately
    const int64_t full = (a.nx % 4 == 0) ? a.nx / K8_TX : 0;
    const int64_t total = (a.nx + K8_TX - 1) / K8_TX;
    if (full > 0) {
        a.xt0 = 0;
        dim3 grid((unsigned)full, gy, gz);
        if (same) k_step3d<RULE, true, true><<<grid, block, dyn, st>>>(a, rx, ry, rz);
        else k_step3d<RULE, false, true><<<grid, block, dyn, st>>>(a, rx, ry, rz);
    }
    if (total > full) {
        a.xt0 = full;
        dim3 grid((unsigned)(total - full), gy, gz);
        if (same) k_step3d<RULE, true, false><<<grid, block, dyn, st>>>(a, rx, ry, rz);
        else k_step3d<RULE, false, false><<<grid, block, dyn, st>>>(a, rx, ry, rz);
    }
    return cudaGetLastError();
}

int64_t step3d_zchunk(int64_t nx, int64_t ny, int64_t nz)
{
    const int64_t tiles = ((nx + K8_TX - 1) / K8_TX) * ((ny + K8_TY - 1) / K8_TY);
#ifndef FQNM_K8_CTAS_PER_SM
#define FQNM_K8_CTAS_PER_SM 12
#endif
#ifndef FQNM_K8_ZMAX
#define FQNM_K8_ZMAX 128
#endif
    int64_t zc = tiles * nz / (148 * FQNM_K8_CTAS_PER_SM);   // ~12 CTAs per SM in total
    if (zc < 16) zc = 16;
    if (zc > FQNM_K8_ZMAX) zc = FQNM_K8_ZMAX;
    if (zc >= nz) return nz;
    // equal chunks (no short last chunk: 512 planes in chunks of 73 left one of 1 plane)
    const int64_t nch = (nz + zc - 1) / zc;
    return (nz + nch - 1) / nch;
}

cudaError_t launch_step3d(int rule, bool same, const Step3DArgs& a, const DevRule& rx,
                          const DevRule& ry, const DevRule& rz, cudaStream_t st)
{
    if (a.zchunk < 1) return cudaErrorInvalidValue;
    switch (rule) {
        case R_LIN_HALF: return step3d_rule<R_LIN_HALF>(same, a, rx, ry, rz, st);
        case R_EO_FAST: return step3d_rule<R_EO_FAST>(same, a, rx, ry, rz, st);
        case R_EO_P1: return step3d_rule<R_EO_P1>(same, a, rx, ry, rz, st);
        case R_GENERIC: return step3d_rule<R_GENERIC>(same, a, rx, ry, rz, st);
        case R_LIN_FAST: return step3d_rule<R_LIN_FAST>(same, a, rx, ry, rz, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fqnm
