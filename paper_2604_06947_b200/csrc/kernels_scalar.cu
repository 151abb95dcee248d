// Scalar FQNM kernels for sm_100a (B200).
//
// The update:
//   F_{i+1/2} = phi+(q_i) + phi-(q_{i+1}),   q_i <- q_i - (F_{i+1/2} - F_{i-1/2})
// is a 3-point integer stencil with no dense contraction, so no tensor cores:
// the design goal is integer-issue throughput with HBM traffic amortised over k
// steps per round trip.
//
//   K1 k_naive            one thread per cell, one step per launch (reference/fallback)
//   K2 k_blocked          temporally blocked: each warp holds a window of 32*V
//                         contiguous cells in registers (V per lane), advances it
//                         k steps with warp shuffles for the neighbour maps, and
//                         stores the cells whose light cone stayed inside the
//                         window (overlapped trapezoids, no smem, no barriers)
//   K3 k_warp_ensemble    one periodic/transmissive problem of 32*V cells per
//                         warp, all nsteps in registers (ensembles, cfg1)
//   K4 k_cta_ensemble     one problem per CTA in shared memory (general small N)
//   +  transfer / min-max / observe helpers
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "fqnm_internal.h"
#include "maps.cuh"

// The launchers are split into parts so the build compiles them as separate
// translation units in parallel (kernels_scalar_p*.cu); part 0 = everything.
#ifndef FQNM_SCALAR_PART
#define FQNM_SCALAR_PART 0
#endif
#define FQNM_PART(x) (FQNM_SCALAR_PART == 0 || FQNM_SCALAR_PART == (x))

#ifndef FQNM_STREAM_STEP
#define FQNM_STREAM_STEP 0     // K2/K3/K6 interior cells updated in map order (variant)
#endif

#ifndef FQNM_RES_LL
#define FQNM_RES_LL 1          // K6 halo exchange in {value, tag} words (no fence / flag round trip)
#endif

#ifndef FQNM_RES_FENCE
#define FQNM_RES_FENCE 0
#endif

namespace fqnm {

static constexpr unsigned FULL = 0xffffffffu;
// spin budget before declaring a peer/neighbour dead: trap (a clean launch
// failure the host sees) instead of hanging the GPU (~20 s at 2 GHz)
static constexpr long long SPIN_TRAP_CYCLES = 40000000000ll;

// ---------------------------------------------------------------------------
// one explicit step of V register-resident cells of a lane, from (g, m) with
// g = phi+ + phi-, m = phi-:  F_{j+1/2} = phi+(q_j) + phi-(q_{j+1}) = g_j - m_j + m_{j+1}.
//   pl, mr: phi+ of the cell left of q[0], phi- of the cell right of q[V-1]
//   WALL:   transmissive ghost rule (interface -1/2 and N-1/2 use the edge cell:
//           F = phi+(q_e) + phi-(q_e) = g_e)
template <int V, bool WALL>
__device__ __forceinline__ void step_cells(int32_t (&q)[V], const int32_t (&g)[V],
                                           const int32_t (&m)[V], int32_t pl, int32_t mr,
                                           int64_t g0, int64_t n)
{
    int32_t Tl = pl + m[0];                 // F_{j-1/2} for j = 0
#pragma unroll
    for (int j = 0; j < V; ++j) {
        int32_t Tr = g[j] - m[j] + ((j + 1 < V) ? m[j + 1] : mr);   // F_{j+1/2}
        if (WALL) {
            if (g0 + j == 0) Tl = g[j];                 // F_{-1/2} with ghost q_{-1} = q_0
            if (g0 + j == n - 1) Tr = g[j];             // F_{N-1/2} with ghost q_N = q_{N-1}
        }
        q[j] = q[j] + Tl - Tr;
        Tl = Tr;
    }
}

template <int RULE, int V>
__device__ __forceinline__ void eval_maps(const int32_t (&q)[V], int32_t (&g)[V],
                                          int32_t (&m)[V], const DevRule& r)
{
#pragma unroll
    for (int j = 0; j < V; j += 2) {          // odd cells may take the other pipe mix
        phi_gm<RULE, false, true>(q[j], g[j], m[j], r);
        if (j + 1 < V) phi_gm<RULE, true, true>(q[j + 1], g[j + 1], m[j + 1], r);
    }
}

// ---------------------------------------------------------------------------
// One explicit step of the lane's V cells.  NB = 0: neighbours by shfl.up/down
// (window edges produce garbage that the caller cuts off); NB = 1: periodic
// wrap inside the warp (K3, the warp holds a whole problem).
//
// SIGN (EO rules, no walls): 1 = every cell of the window has q >= 0, 2 = every cell has
// q <= 0.  By the monotonicity the planner proves (D8: the update is non-decreasing in
// each argument and keeps constants, Lemma CFL) a window whose cells are all
// >= 0 stays >= 0 inside its dependence cone for all k steps, so there phi- = 0 and the
// interface transfer is F_{j+1/2} = phi+(q_j) = g_j; for q <= 0, F_{j+1/2} = phi-(q_{j+1})
// = g_{j+1}.  Cells outside the cone are cut off by the caller either way.
#ifndef FQNM_LIN_STREAM
#define FQNM_LIN_STREAM 0      // LIN kappa = 1/2 step streamed cell by cell (variant)
#endif
#ifndef FQNM_SIGN_STREAM
#define FQNM_SIGN_STREAM 1     // sign-uniform step: maps evaluated cell by cell (no map array)
#endif
// SIGN_ = SIGN + 2 (3, 4): the same sign-uniform steps with the float32 form of the EO
// magnitude (K6: a lone warp per sub-partition is latency-bound, and the float64 form's
// longer latency costs it 5 %)
template <int RULE, int V, bool WALL, int NB, int SIGN_ = 0>
__device__ __forceinline__ void one_step(int32_t (&q)[V], const DevRule& r, int lane, int64_t g0,
                                         int64_t n)
{
    constexpr int SIGN = SIGN_ > 2 ? SIGN_ - 2 : SIGN_;
    constexpr bool F32 = SIGN_ > 2;
    if (FQNM_SIGN_STREAM && SIGN != 0 && !WALL && (RULE == R_EO_P1 || RULE == R_EO_FAST)) {
        // streamed: the lane-edge map first (for the shuffle), then each cell's map right
        // before its update, so the ALU-pipe updates interleave with the map evaluation
        // and no array of maps is live
        if (SIGN == 1) {                   // q_j += g_{j-1} - g_j
            const int32_t glast = eo_g_sel<RULE, true, F32>(q[V - 1], r);
            int32_t gp = NB == 0 ? __shfl_up_sync(FULL, glast, 1)
                                 : __shfl_sync(FULL, glast, (lane + 31) & 31);
#if FQNM_EO_SIGN_CONV != 2 && FQNM_EO_SIGN_LEA != 2
            // every cell evaluates the same form: a plain cell loop (micro: 0.90 vs 0.86 issue
            // for the paired loop below, which alternating variants need)
#pragma unroll
            for (int j = 0; j + 1 < V; ++j) {
                const int32_t gj = eo_g_sel<RULE, false, F32>(q[j], r);
                q[j] = q[j] + gp - gj;
                gp = gj;
            }
#else
#pragma unroll
            for (int j = 0; j + 1 < V; j += 2) {         // V even: j + 1 <= V - 2 here
                const int32_t g0 = eo_g_sel<RULE, false, F32>(q[j], r);
                q[j] = q[j] + gp - g0;
                if (j + 2 < V) {
                    const int32_t g1 = eo_g_sel<RULE, true, F32>(q[j + 1], r);
                    q[j + 1] = q[j + 1] + g0 - g1;
                    gp = g1;
                } else {
                    gp = g0;
                }
            }
#endif
            q[V - 1] = q[V - 1] + gp - glast;
        } else {                           // q_j += g_j - g_{j+1}
            const int32_t g0 = eo_g_sel<RULE, false, F32>(q[0], r);
            const int32_t gr = NB == 0 ? __shfl_down_sync(FULL, g0, 1)
                                       : __shfl_sync(FULL, g0, (lane + 1) & 31);
            int32_t gc = g0;
#pragma unroll
            for (int j = 0; j + 1 < V; j += 2) {
                const int32_t g1 = eo_g_sel<RULE, true, F32>(q[j + 1], r);
                q[j] = q[j] + gc - g1;
                gc = g1;
                if (j + 2 < V) {
                    const int32_t g2 = eo_g_sel<RULE, false, F32>(q[j + 2], r);
                    q[j + 1] = q[j + 1] + gc - g2;
                    gc = g2;
                }
            }
            q[V - 1] = q[V - 1] + gc - gr;
        }
    } else if (SIGN != 0 && !WALL && (RULE == R_EO_P1 || RULE == R_EO_FAST)) {
        int32_t g[V];
#pragma unroll
        for (int j = 0; j < V; j += 2) {
            g[j] = eo_g_sel<RULE, false, F32>(q[j], r);
            if (j + 1 < V) g[j + 1] = eo_g_sel<RULE, true, F32>(q[j + 1], r);
        }
        if (SIGN == 1) {                   // q_j += g_{j-1} - g_j
            const int32_t gl = NB == 0 ? __shfl_up_sync(FULL, g[V - 1], 1)
                                       : __shfl_sync(FULL, g[V - 1], (lane + 31) & 31);
            q[0] = q[0] + gl - g[0];
#pragma unroll
            for (int j = 1; j < V; ++j) q[j] = q[j] + g[j - 1] - g[j];
        } else {                           // q_j += g_j - g_{j+1}
            const int32_t gr = NB == 0 ? __shfl_down_sync(FULL, g[0], 1)
                                       : __shfl_sync(FULL, g[0], (lane + 1) & 31);
#pragma unroll
            for (int j = 0; j + 1 < V; ++j) q[j] = q[j] + g[j] - g[j + 1];
            q[V - 1] = q[V - 1] + g[V - 1] - gr;
        }
    } else if ((FQNM_LIN_STREAM || V > 32) && RULE == R_LIN_HALF && !WALL) {
        // kappa = 1/2 streamed: phi+ of the lane's last cell first (for the shuffle),
        // then cell by cell h_j = trunc(q_j/2), q'_j = phi+(q_{j-1}) + h_j (no arrays)
        const int32_t hl = q[V - 1] / 2;
        const int32_t plast = hl * r.mone + q[V - 1];
        int32_t pp = NB == 0 ? __shfl_up_sync(FULL, plast, 1)
                             : __shfl_sync(FULL, plast, (lane + 31) & 31);
#pragma unroll
        for (int j = 0; j + 1 < V; ++j) {
            const int32_t h = q[j] / 2;
            const int32_t p = h * r.mone + q[j];
            q[j] = pp * r.one + h;
            pp = p;
        }
        q[V - 1] = pp * r.one + hl;
    } else if (RULE == R_LIN_HALF && !WALL) {
        // kappa = 1/2: q'_j = trunc(q_j/2) + phi+(q_{j-1}), phi+ = q - trunc(q/2).
        // The runtime r.one turns the two adds into IMADs (FMA pipe) so the
        // ALU pipe only carries the halving (LEA.HI + SHF): 2 ALU + 2 FMA ops.
        int32_t h[V], p[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            h[j] = q[j] / 2;
            p[j] = h[j] * r.mone + q[j];
        }
        const int32_t pl = NB == 0 ? __shfl_up_sync(FULL, p[V - 1], 1)
                                   : __shfl_sync(FULL, p[V - 1], (lane + 31) & 31);
        q[0] = pl * r.one + h[0];
#pragma unroll
        for (int j = 1; j < V; ++j) q[j] = p[j - 1] * r.one + h[j];
    } else if (RULE == R_TWOPOINT || RULE == R_TP_FAST) {
        // two-point rule: T_{j+1/2} = Phi(q_j, q_{j+1}); needs the right neighbour's state
        const int32_t qr = NB == 0 ? __shfl_down_sync(FULL, q[0], 1)
                                   : __shfl_sync(FULL, q[0], (lane + 1) & 31);
        int32_t T[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            int32_t qn = (j + 1 < V) ? q[j + 1] : qr;
            if (WALL && g0 + j == n - 1) qn = q[j];             // ghost q_N = q_{N-1}
            T[j] = tp_eval<RULE>(q[j], qn, r);
        }
        int32_t Tl = NB == 0 ? __shfl_up_sync(FULL, T[V - 1], 1)
                             : __shfl_sync(FULL, T[V - 1], (lane + 31) & 31);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            if (WALL && g0 + j == 0) Tl = tp_eval<RULE>(q[j], q[j], r);  // ghost q_{-1} = q_0
            const int32_t t = T[j];
            q[j] = q[j] + Tl - t;
            Tl = t;
        }
    } else if (FQNM_STREAM_STEP && NB == 0 && !WALL && V >= 4) {
        // interior cells first, in cell order: the maps of cell j+1 are evaluated right
        // before cell j is updated (FMA-pipe map work interleaved with the ALU-pipe
        // updates); the two cells that need the neighbour lanes' maps come last, after
        // the shuffles
        int32_t g[V], m[V];
        phi_gm<RULE, false, true>(q[0], g[0], m[0], r);
        phi_gm<RULE, true, true>(q[1], g[1], m[1], r);
        const int32_t q0 = q[0];
        int32_t Tl = g[0] - m[0] + m[1];                                // F_{1/2}
#pragma unroll
        for (int j = 1; j + 1 < V; ++j) {
            if (j & 1) phi_gm<RULE, false, true>(q[j + 1], g[j + 1], m[j + 1], r);
            else phi_gm<RULE, true, true>(q[j + 1], g[j + 1], m[j + 1], r);
            const int32_t Tr = g[j] - m[j] + m[j + 1];                  // F_{j+1/2}
            q[j] = q[j] + Tl - Tr;
            Tl = Tr;
        }
        const int32_t pl = __shfl_up_sync(FULL, g[V - 1] - m[V - 1], 1);
        const int32_t mr = __shfl_down_sync(FULL, m[0], 1);
        q[0] = q0 + (pl + m[0]) - (g[0] - m[0] + m[1]);
        q[V - 1] = q[V - 1] + Tl - (g[V - 1] - m[V - 1] + mr);
    } else {
        int32_t g[V], m[V];
        eval_maps<RULE, V>(q, g, m, r);
        const int32_t pv = g[V - 1] - m[V - 1];
        const int32_t pl = NB == 0 ? __shfl_up_sync(FULL, pv, 1)
                                   : __shfl_sync(FULL, pv, (lane + 31) & 31);
        const int32_t mr = NB == 0 ? __shfl_down_sync(FULL, m[0], 1)
                                   : __shfl_sync(FULL, m[0], (lane + 1) & 31);
        step_cells<V, WALL>(q, g, m, pl, mr, g0, n);
    }
}

#ifndef FQNM_FUSED_STEPS
#define FQNM_FUSED_STEPS 0     // K2 fast path: interleave step s's update with step s+1's maps
                               // (measured slower: EO 2416 vs 2477, LIN 6112 vs 6349 GCUPS)
#endif

// One fused step (no walls, neighbours by shfl): update the lane's cells with the
// current maps (g, m) and, cell by cell, evaluate the maps of the new value for the
// next step (NEXT).  Interleaving the ALU-heavy update with the FMA-heavy map
// evaluation keeps both pipes busy instead of running the step in pipe phases.
template <int RULE, int V, bool NEXT>
__device__ __forceinline__ void fused_step(int32_t (&q)[V], int32_t (&g)[V], int32_t (&m)[V],
                                           const DevRule& r)
{
    const int32_t pl = __shfl_up_sync(FULL, g[V - 1] - m[V - 1], 1);
    const int32_t mr = __shfl_down_sync(FULL, m[0], 1);
    int32_t Tl = pl + m[0];                                         // F_{-1/2} of the lane
#pragma unroll
    for (int j = 0; j < V; j += 2) {          // odd cells may take the other pipe mix
        int32_t Tr = g[j] - m[j] + ((j + 1 < V) ? m[j + 1] : mr);         // F_{j+1/2}
        q[j] = q[j] + Tl - Tr;
        Tl = Tr;
        if (NEXT) phi_gm<RULE, false, true>(q[j], g[j], m[j], r);
        if (j + 1 < V) {
            Tr = g[j + 1] - m[j + 1] + ((j + 2 < V) ? m[j + 2] : mr);
            q[j + 1] = q[j + 1] + Tl - Tr;
            Tl = Tr;
            if (NEXT) phi_gm<RULE, true, true>(q[j + 1], g[j + 1], m[j + 1], r);
        }
    }
}

template <int V, bool NEXT>
__device__ __forceinline__ void fused_step_lin_half(int32_t (&q)[V], int32_t (&h)[V],
                                                    int32_t (&p)[V], const DevRule& r)
{
    // kappa = 1/2: q'_j = trunc(q_j/2) + phi+(q_{j-1}) with h = trunc(q/2), p = q - h
    int32_t pprev = __shfl_up_sync(FULL, p[V - 1], 1);
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int32_t pj = p[j];
        q[j] = pprev * r.one + h[j];
        pprev = pj;
        if (NEXT) {
            h[j] = q[j] / 2;
            p[j] = h[j] * r.mone + q[j];
        }
    }
}

// K2: temporally blocked stencil
template <int RULE, int V, bool WALL, int SIGN = 0>
__device__ __forceinline__ void run_window_steps(int32_t (&q)[V], int ksteps, const DevRule& r,
                                                 int64_t g0, int64_t n)
{
    const int lane = threadIdx.x & 31;
    if (SIGN != 0) {
        int s = 0;
        for (; s + 2 <= ksteps; s += 2) {
            one_step<RULE, V, WALL, 0, SIGN>(q, r, lane, g0, n);
            one_step<RULE, V, WALL, 0, SIGN>(q, r, lane, g0, n);
        }
        if (s < ksteps) one_step<RULE, V, WALL, 0, SIGN>(q, r, lane, g0, n);
        return;
    }
    if (FQNM_FUSED_STEPS && RULE != R_TWOPOINT && RULE != R_TP_FAST && !WALL && ksteps > 0) {
        int32_t g[V], m[V];
        if (RULE == R_LIN_HALF) {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                g[j] = q[j] / 2;
                m[j] = g[j] * r.mone + q[j];
            }
        } else {
            eval_maps<RULE, V>(q, g, m, r);
        }
        int s = 1;
        for (; s + 2 <= ksteps; s += 2) {
            if (RULE == R_LIN_HALF) {
                fused_step_lin_half<V, true>(q, g, m, r);
                fused_step_lin_half<V, true>(q, g, m, r);
            } else {
                fused_step<RULE, V, true>(q, g, m, r);
                fused_step<RULE, V, true>(q, g, m, r);
            }
        }
        if (s < ksteps) {
            if (RULE == R_LIN_HALF) fused_step_lin_half<V, true>(q, g, m, r);
            else fused_step<RULE, V, true>(q, g, m, r);
        }
        if (RULE == R_LIN_HALF) fused_step_lin_half<V, false>(q, g, m, r);
        else fused_step<RULE, V, false>(q, g, m, r);
        return;
    }
    int s = 0;
    // unrolled by two: no register renaming moves between steps
    for (; s + 2 <= ksteps; s += 2) {
        one_step<RULE, V, WALL, 0>(q, r, lane, g0, n);
        one_step<RULE, V, WALL, 0>(q, r, lane, g0, n);
    }
    if (s < ksteps) one_step<RULE, V, WALL, 0>(q, r, lane, g0, n);
}

#ifndef FQNM_SIGN_WINDOWS
#define FQNM_SIGN_WINDOWS 1    // K2/K2P/K6 EO: sign-uniform windows step on g alone (one_step SIGN)
#endif

// k steps of a window without walls (neighbours by shfl, edges cut off by the caller).
// EO rules: one warp vote per window on the sign of its cells picks the sign-uniform
// step (one_step SIGN) where it applies
template <int RULE, int V, bool F32 = false>
__device__ __forceinline__ void run_window_steps_signed(int32_t (&q)[V], int ksteps,
                                                        const DevRule& r)
{
#ifdef FQNM_FORCE_SIGN
    // experiment builds only: every window taken as sign-uniform (valid for such data only)
    if (RULE == R_EO_P1 || RULE == R_EO_FAST) {
        run_window_steps<RULE, V, false, FQNM_FORCE_SIGN>(q, ksteps, r, 0, 0);
        return;
    }
#endif
    if (FQNM_SIGN_WINDOWS && RULE == R_TP_FAST) {
        // Godunov for Burgers, Phi(qL, qR) = g(max(max(qL, 0), -min(qR, 0))) with the EO
        // magnitude map g (even in q): on a window whose cells are all >= 0 it is g(qL), on
        // one whose cells are all <= 0 it is g(qR) -- exactly the split EO rule's transfer
        // there (the collapse of Thm transfer-operator equivalence), so such
        // windows take the EO sign-uniform step (7 instructions per cell-update instead of
        // the two-point evaluation).  Godunov is monotone on the D8 range (DESIGN A18), so
        // the sign holds for the k steps on the dependence cone, as for EO.
        int32_t lo = q[0], hi = q[0];
#pragma unroll
        for (int j = 1; j < V; ++j) { lo = min(lo, q[j]); hi = max(hi, q[j]); }
        const bool pos = __all_sync(FULL, lo >= 0);
        if (pos || __all_sync(FULL, hi <= 0)) {
            if (r.tp_fast == 1) {
                if (pos) run_window_steps<R_EO_P1, V, false, 1>(q, ksteps, r, 0, 0);
                else run_window_steps<R_EO_P1, V, false, 2>(q, ksteps, r, 0, 0);
            } else {
                if (pos) run_window_steps<R_EO_FAST, V, false, 1>(q, ksteps, r, 0, 0);
                else run_window_steps<R_EO_FAST, V, false, 2>(q, ksteps, r, 0, 0);
            }
            return;
        }
    }
    if (FQNM_SIGN_WINDOWS && (RULE == R_EO_P1 || RULE == R_EO_FAST)) {
        int32_t lo = q[0], hi = q[0];
#pragma unroll
        for (int j = 1; j < V; ++j) { lo = min(lo, q[j]); hi = max(hi, q[j]); }
        if (__all_sync(FULL, lo >= 0)) { run_window_steps<RULE, V, false, F32 ? 3 : 1>(q, ksteps, r, 0, 0); return; }
        if (__all_sync(FULL, hi <= 0)) { run_window_steps<RULE, V, false, F32 ? 4 : 2>(q, ksteps, r, 0, 0); return; }
    }
    run_window_steps<RULE, V, false>(q, ksteps, r, 0, 0);
}

__device__ __forceinline__ int64_t wrap_index(int64_t i, int64_t n, int bmode, int64_t halo)
{
    if (bmode == BM_PERIODIC) {
        i %= n;
        return i < 0 ? i + n : i;
    }
    if (bmode == BM_TRANSMISSIVE) return i < 0 ? 0 : (i >= n ? n - 1 : i);
    // HALO: buffer index = i + halo, valid range [-halo, n + halo)
    if (i < -halo) i = -halo;
    if (i >= n + halo) i = n + halo - 1;
    return i + halo;
}

// ---- fused peer-memory halo exchange (split domains over NVLink) ----------
__device__ __forceinline__ void p2p_wait(const unsigned int* flag, uint32_t tag)
{
    unsigned int f;
    const long long t0 = clock64();
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
        if ((int)(f - tag) >= 0) break;
        if (clock64() - t0 > SPIN_TRAP_CYCLES) __trap();
    }
}

__device__ __forceinline__ void p2p_signal(unsigned int* flag, uint32_t tag)
{
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(flag), "r"(tag) : "memory");
}

// push the H edge cells of `ext` (layout [H | n | H]) that `owned0` / the window
// covers into the neighbours' buffers and release `tag` on their flags
static __device__ __noinline__ void p2p_push(const BlockedArgs& a, const int32_t* ext, bool left_edge,
                                      bool right_edge, uint32_t tag, int32_t* peer_l,
                                      int32_t* peer_r, int lane)
{
    const int64_t H = a.halo, n = a.n;
    if (left_edge) {            // my [0, H) -> left neighbour's right halo [H + left_n, ...)
        for (int64_t i = lane; i < H; i += 32) peer_l[H + a.left_n + i] = ext[H + i];
        __threadfence_system();
        __syncwarp();
        if (lane == 0) p2p_signal(a.peer_left_flags + 1, tag);
    }
    if (right_edge) {           // my [n - H, n) -> right neighbour's left halo [0, H)
        for (int64_t i = lane; i < H; i += 32) peer_r[i] = ext[n + i];
        __threadfence_system();
        __syncwarp();
        if (lane == 0) p2p_signal(a.peer_right_flags + 0, tag);
    }
    __syncwarp();
}

// initial halos of a split run: every rank pushes the edges of its current buffer
static __global__ void k_halo_prime(BlockedArgs a)
{
    const int lane = threadIdx.x & 31;
    p2p_push(a, a.src, true, true, a.tag, a.peer_left_dst, a.peer_right_dst, lane);
}

#if FQNM_PART(1)
cudaError_t launch_halo_prime(const BlockedArgs& a, cudaStream_t st)
{
    k_halo_prime<<<1, 32, 0, st>>>(a);
    return cudaGetLastError();
}

#endif  // part 1

// Slow window (periodic wrap, transmissive walls, ragged tails, misaligned
// batches): scalar loads through wrap_index, guarded scalar stores.  Kept out of
// line so the hot path's register allocation is not shaped by it.
template <int RULE, int V>
__device__ __noinline__ void slow_window(const BlockedArgs& a, const DevRule& r, int64_t b,
                                         int64_t ws, int lane)
{
    constexpr int W = 32 * V;
    const int64_t n = a.n;
    const int64_t pstride = (a.bmode == BM_HALO) ? n + 2 * a.halo : n;
    const int32_t* src = a.src + b * pstride;
    int32_t* dst = a.dst + b * pstride + ((a.bmode == BM_HALO) ? a.halo : 0);
    const int64_t g0 = ws + lane * V;
    int32_t q[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int32_t* x = src + wrap_index(g0 + j, n, a.bmode, a.halo);
        q[j] = a.p2p ? __ldcg(x) : *x;          // p2p: halos written by a peer in this launch
    }
    if (a.bmode == BM_TRANSMISSIVE)
        run_window_steps<RULE, V, true>(q, a.ksteps, r, g0, n);
    else
        run_window_steps<RULE, V, false>(q, a.ksteps, r, g0, n);
    const int lo = a.KL, hi = W - a.KR;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int pos = lane * V + j;
        const int64_t gi = g0 + j;
        if (pos >= lo && pos < hi && gi >= 0 && gi < n) dst[gi] = q[j];
    }
}


#ifndef FQNM_PREFETCH
#define FQNM_PREFETCH 0        // K2: stage the next window in shared memory (cp.async) while stepping
                               // (measured 2.3% slower at V = 32: the staging registers spill)
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa), "l"(gmem) : "memory");
}

// FSIGN (K2S, EO rules): 0 = vote per window (general K2), 1 = every cell >= 0, 2 = every
// cell <= 0 for the whole call (host-proved from the range check's min/max, or the dual
// launch's sign_bits): the fast windows step with one_step SIGN directly
template <int RULE, int V, int MINB, int FSIGN = 0>
__global__ void __launch_bounds__(256, MINB) k_blocked(BlockedArgs a, DevRule r)
{
    static_assert(V % 4 == 0, "V must be a multiple of 4 (int4 vectors)");
    if (a.guard && *a.guard) return;                            // input failed its range check
    if (a.sign_bits) {                                          // dual launch: one of the two runs
        const bool has_neg = (*a.sign_bits & 1) != 0;
        if (FSIGN == 1 ? has_neg : !has_neg) return;
    }
    constexpr int W = 32 * V;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int S = W - a.KL - a.KR;
    const int lo = a.KL, hi = W - a.KR;
    const int64_t n = a.n;
    const bool halo = a.bmode == BM_HALO;
    const int64_t pstride = halo ? n + 2 * a.halo : n;
    const int64_t lowest = halo ? -a.halo : 0;
#if FQNM_PREFETCH
    // per warp: the next window's 32*V cells as [V/4][32 lanes] int4 (conflict-free LDS.128)
    __shared__ int4 stage[256 / 32][V / 4][32];
    int4 (&my)[V / 4][32] = stage[threadIdx.x >> 5];
    bool staged = false;
#endif
    // window geometry of (b, w): first cell ws, problem offset boff, fast = int4 path
    auto geom = [&](int64_t bb, int64_t ww, int64_t& ws, int64_t& boff, int64_t& owned0) {
        owned0 = ww * S;
        if (a.p2p && owned0 + S > n && n >= S) owned0 = n - S;  // last window ends at n
        ws = owned0 - a.KL;                                     // first cell of the window
        boff = bb * pstride + (halo ? a.halo : 0);
        return ((boff & 3) == 0) && ws >= lowest && ws + W <= n;
    };
    // window iteration without 64-bit division: (b, w) advanced by nwarps
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t b = 0;
    while (w >= a.nwin && b < a.batch) { w -= a.nwin; ++b; }
    while (b < a.batch) {
        int64_t ws, boff, owned0;
        const bool fast = geom(b, w, ws, boff, owned0);
        if (a.p2p && (ws < 0 || ws + W > n)) {                  // reads halos: wait for them
            if (lane == 0) {
                if (ws < 0) p2p_wait(a.self_flags + 0, a.tag);
                if (ws + W > n) p2p_wait(a.self_flags + 1, a.tag);
            }
            __syncwarp();
        }
        int64_t w2 = w + nwarps, b2 = b;
        while (w2 >= a.nwin && b2 < a.batch) { w2 -= a.nwin; ++b2; }
        if (fast) {
            int4* d4 = reinterpret_cast<int4*>(a.dst + boff + ws) + lane * (V / 4);
            int32_t q[V];
#if FQNM_PREFETCH
            if (staged) {
                asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
                for (int j = 0; j < V / 4; ++j) {
                    const int4 v = my[j][lane];
                    q[4 * j] = v.x; q[4 * j + 1] = v.y; q[4 * j + 2] = v.z; q[4 * j + 3] = v.w;
                }
            } else
#endif
            {
                const int4* s4 = reinterpret_cast<const int4*>(a.src + boff + ws) + lane * (V / 4);
                if (a.p2p && ws < 0) {
                    // the left halo was written by the peer GPU during this launch (released
                    // by its flag): coherent L2 loads, not the read-only path
#pragma unroll
                    for (int j = 0; j < V / 4; ++j) {
                        int4 v = __ldcg(s4 + j);
                        q[4 * j] = v.x; q[4 * j + 1] = v.y; q[4 * j + 2] = v.z; q[4 * j + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < V / 4; ++j) {
                        int4 v = __ldg(s4 + j);
                        q[4 * j] = v.x; q[4 * j + 1] = v.y; q[4 * j + 2] = v.z; q[4 * j + 3] = v.w;
                    }
                }
            }
#if FQNM_PREFETCH
            // stage the next window (fast, and not a halo window of a p2p run, whose
            // halos may not have arrived yet) while this one steps
            staged = false;
            if (b2 < a.batch) {
                int64_t ws2, boff2, o2;
                if (geom(b2, w2, ws2, boff2, o2) && !(a.p2p && (ws2 < 0 || ws2 + W > n))) {
                    const int4* s4n = reinterpret_cast<const int4*>(a.src + boff2 + ws2) + lane * (V / 4);
#pragma unroll
                    for (int j = 0; j < V / 4; ++j) cp_async16(&my[j][lane], s4n + j);
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    staged = true;
                }
            }
#endif
            if (FSIGN != 0) run_window_steps<RULE, V, false, FSIGN>(q, a.ksteps, r, 0, 0);
            else run_window_steps_signed<RULE, V>(q, a.ksteps, r);
            // store the cells whose dependence cone stayed inside the window
#pragma unroll
            for (int j = 0; j < V / 4; ++j) {
                const int pos = lane * V + 4 * j;
                if (pos >= lo && pos < hi)
                    d4[j] = make_int4(q[4 * j], q[4 * j + 1], q[4 * j + 2], q[4 * j + 3]);
            }
        } else {
            slow_window<RULE, V>(a, r, b, ws, lane);
#if FQNM_PREFETCH
            staged = false;
#endif
        }
        if (a.p2p && (owned0 == 0 || owned0 + S >= n)) {
            __syncwarp();
            p2p_push(a, a.dst, owned0 == 0, owned0 + S >= n, a.tag + 1, a.peer_left_dst,
                     a.peer_right_dst, lane);
        }
        w = w2;
        b = b2;
    }
#if FQNM_PREFETCH
    asm volatile("cp.async.wait_all;" ::: "memory");
#endif
}

// ---------------------------------------------------------------------------
// K2P: persistent K2.  One launch runs all nblocks blocks of k steps: warps claim items
// (block b, window w) in increasing order from a global counter; an item of block b > 0
// first acquires the flags of the block b-1 windows whose owned cells overlap its input
// window (they are earlier items, claimed by running warps, so the wait always ends),
// then steps the window exactly as K2 and releases its own flag.  Loads bypass L1
// (ld.global.cg): the inputs were written inside this launch by other SMs.  The wait
// set is widened symmetrically (max(KL, KR) on both sides) so it also orders the
// write-after-read on the ping-pong buffer (see persist_wait_cover).
// Removes the per-launch tail (the last partial wave of windows) and launch gaps.
// Wait for the block b-1 windows whose owned cells overlap [wS - E, wS + S + E),
// E = max(KL, KR) (periodic wrap / clamped walls): they cover the item's input window
// (read after write) and include every block b-1 item that reads the cells this item
// overwrites in the other buffer (write after read: those items' input windows reach
// KL/KR cells into this window's owned range).  The whole warp takes part (lane i
// polls the i-th window) so it never diverges around the hot loop; relaxed polling,
// one acquire fence at the end.
// the window this lane polls for item (b, w), or -1: lanes 0..2 take w-1, w, w+1 when the
// widened range fits in the neighbours (E <= S, the usual case), else the general cover
static __device__ __forceinline__ int64_t persist_cover_window(const PersistArgs& a, int64_t w, int lane)
{
    const int64_t n = a.n, S = a.S, nwin = a.nwin;
    const int64_t E = a.KL > a.KR ? a.KL : a.KR;
    int64_t my = -1;
    if (E <= S && nwin >= 4) {
        // [wS - E, wS + S + E) touches windows w-1, w, w+1 only; at the periodic wrap the
        // last window may be short, so its left neighbour is covered too
        if (lane < 3) {
            my = w - 1 + lane;
            if (a.bmode == BM_PERIODIC) my = my < 0 ? my + nwin : (my >= nwin ? my - nwin : my);
            else my = my < 0 ? 0 : (my >= nwin ? nwin - 1 : my);
        } else if (lane == 3 && a.bmode == BM_PERIODIC) {
            // a short last window: the range of w = 0 reaches back into window nwin - 2, and
            // the ranges of the last two windows reach forward into window 0
            if (w == 0) my = nwin - 2;
            else if (w >= nwin - 2) my = 0;
        }
        return my;
    }
    const int64_t span = (S + 2 * E + S - 1) / S + 1;          // windows touched, upper bound
    const int64_t lo = w * S - E, hi = w * S + S + E - 1;
    if (lane < 2 * span + 2) {
        int64_t x = lo + (int64_t)lane * S;
        if (x > hi) x = hi;
        if (a.bmode == BM_PERIODIC) { x %= n; if (x < 0) x += n; }
        else x = x < 0 ? 0 : (x >= n ? n - 1 : x);
        my = x / S;
        if (my >= nwin) my = nwin - 1;
    }
    if (lane == 31 && a.bmode == BM_PERIODIC && (lo < 0 || hi >= n)) my = nwin - 1 > 0 ? nwin - 2 : 0;
    if (lane == 30 && a.bmode == BM_PERIODIC && (lo < 0 || hi >= n)) my = nwin - 1;
    return my;
}

// one relaxed poll of the lane's window flag: true when it carries at least `target`
static __device__ __forceinline__ bool persist_poll(const PersistArgs& a, int64_t my, uint32_t target)
{
    if (my < 0) return true;
    unsigned int f;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.flags + my) : "memory");
    return (int)(f - target) >= 0;
}

// Wait for the block b-1 windows whose owned cells overlap [wS - E, wS + S + E),
// E = max(KL, KR) (periodic wrap / clamped walls): they cover the item's input window
// (read after write) and include every block b-1 item that reads the cells this item
// overwrites in the other buffer (write after read: those items' input windows reach
// KL/KR cells into this window's owned range).  The whole warp takes part so it never
// diverges around the hot loop; relaxed polling, one acquire fence at the end.
static __device__ __forceinline__ void persist_wait_cover(const PersistArgs& a, int64_t w,
                                                          uint32_t target, int lane)
{
    const int64_t my = persist_cover_window(a, w, lane);
    const long long t0 = clock64();
    for (;;) {
        if (__all_sync(0xffffffffu, persist_poll(a, my, target))) break;
        if (clock64() - t0 > SPIN_TRAP_CYCLES) __trap();
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");   // acquire: the relaxed reads above
}

// windows that wrap or touch a wall: scalar L1-bypassing loads through wrap_index
template <int RULE, int V>
static __device__ __noinline__ void persist_slow(const int32_t* src, int32_t* dst, int64_t ws,
                                                 int64_t n, int bmode, int ks, const DevRule& r,
                                                 int lo, int hi, int lane)
{
    const int64_t g0 = ws + lane * V;
    int32_t q[V];
#pragma unroll
    for (int j = 0; j < V; ++j) q[j] = __ldcg(src + wrap_index(g0 + j, n, bmode, 0));
    if (bmode == BM_TRANSMISSIVE) run_window_steps<RULE, V, true>(q, ks, r, g0, n);
    else run_window_steps<RULE, V, false>(q, ks, r, g0, n);
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int pos = lane * V + j;
        const int64_t gi = g0 + j;
        if (pos >= lo && pos < hi && gi >= 0 && gi < n) __stcg(dst + gi, q[j]);
    }
}

#ifndef FQNM_K2P_LIN_V
#define FQNM_K2P_LIN_V 48      // cells per lane of the persistent LIN 1/2 kernel (streamed step,
                               // 128 registers): cfg3 7.06 vs 6.96 TCUPS with V = 32
#endif

// FSIGN as k_blocked (K2S): the host proved the whole state >= 0 (1) or <= 0 (2)
template <int RULE, int V, int MINB, int FSIGN = 0>
__global__ void __launch_bounds__(256, MINB) k_blocked_persist(PersistArgs a, DevRule r)
{
    if (a.guard && *a.guard) return;                            // input failed its range check
    if (a.sign_bits) {                                          // dual launch: one of the two runs
        const bool has_neg = (*a.sign_bits & 1) != 0;
        if (FSIGN == 1 ? has_neg : !has_neg) return;
    }
    constexpr int W = 32 * V;
    const int lane = threadIdx.x & 31;
    const int64_t n = a.n, nwin = a.nwin, S = a.S;
    const unsigned long long total = (unsigned long long)a.nblocks * (unsigned long long)nwin;
    const int lo = a.KL, hi = W - a.KR;
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(a.counter, 1ull);
    item = __shfl_sync(FULL, item, 0);
    while (item < total) {
        const int b = (int)(item / (unsigned long long)nwin);
        const int64_t w = (int64_t)(item - (unsigned long long)b * (unsigned long long)nwin);
        const int64_t ws = w * S - a.KL;                           // first cell of the window
        const int32_t* src = (b & 1) ? a.buf1 : a.buf0;
        int32_t* dst = (b & 1) ? a.buf0 : a.buf1;
#ifndef FQNM_PERSIST_NOWAIT
        if (b > 0) persist_wait_cover(a, w, a.tag_base + (uint32_t)b, lane);
#endif
        const int ks = a.base + (b < a.rem ? 1 : 0);
        int32_t q[V];
        if (ws >= 0 && ws + W <= n) {
            const int4* s4 = reinterpret_cast<const int4*>(src + ws) + lane * (V / 4);
#pragma unroll
            for (int j = 0; j < V / 4; ++j) {
                const int4 v = __ldcg(s4 + j);
                q[4 * j] = v.x; q[4 * j + 1] = v.y; q[4 * j + 2] = v.z; q[4 * j + 3] = v.w;
            }
            if (FSIGN != 0) run_window_steps<RULE, V, false, FSIGN>(q, ks, r, 0, 0);
            else run_window_steps_signed<RULE, V>(q, ks, r);
            int4* d4 = reinterpret_cast<int4*>(dst + ws) + lane * (V / 4);
#pragma unroll
            for (int j = 0; j < V / 4; ++j) {
                const int pos = lane * V + 4 * j;
                if (pos >= lo && pos < hi)
                    __stcg(d4 + j, make_int4(q[4 * j], q[4 * j + 1], q[4 * j + 2], q[4 * j + 3]));
            }
        } else {
            persist_slow<RULE, V>(src, dst, ws, n, a.bmode, ks, r, lo, hi, lane);
        }
        // release: every lane fences its own stores (one warp-wide MEMBAR; measured 2-10 %
        // faster than lane 0 fencing for the warp after a warp barrier), then the flag
        __syncwarp();
        __threadfence();
        if (lane == 0) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;"
                         :: "l"(a.flags + w), "r"(a.tag_base + (uint32_t)b + 1u) : "memory");
            item = atomicAdd(a.counter, 1ull);
        }
        item = __shfl_sync(FULL, item, 0);
    }
}

#if FQNM_PART(5)
bool blocked_persist_has_rule(int rule)
{
    return rule == R_LIN_HALF || rule == R_EO_P1 || rule == R_EO_FAST || rule == R_LIN_FAST;
}

// cells per lane of the persistent kernel: the sign-specialised EO variant (sign = 1, 2)
// has the K2S geometry
int blocked_persist_V(int rule, int sign)
{
    if (sign != 0 && (rule == R_EO_P1 || rule == R_EO_FAST)) return BLOCKED_SIGN_V;
    return rule == R_LIN_HALF ? FQNM_K2P_LIN_V : 32;
}

template <int RULE, int V = 32, int FSIGN = 0>
static cudaError_t persist_rule(const PersistArgs& a, const DevRule& r, cudaStream_t st)
{
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, k_blocked_persist<RULE, V, 2, FSIGN>, 256, 0);
    if (e != cudaSuccess) return e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    k_blocked_persist<RULE, V, 2, FSIGN><<<per_sm * sms, 256, 0, st>>>(a, r);
    return cudaGetLastError();
}

cudaError_t launch_blocked_persist(int rule, int sign, const PersistArgs& a, const DevRule& r,
                                   cudaStream_t st)
{
    if (sign != 0) {                                    // K2PS: persistent + sign-specialised
        constexpr int V = BLOCKED_SIGN_V;
        if (rule == R_EO_P1)
            return sign == 1 ? persist_rule<R_EO_P1, V, 1>(a, r, st) : persist_rule<R_EO_P1, V, 2>(a, r, st);
        if (rule == R_EO_FAST)
            return sign == 1 ? persist_rule<R_EO_FAST, V, 1>(a, r, st) : persist_rule<R_EO_FAST, V, 2>(a, r, st);
        return cudaErrorInvalidValue;
    }
    switch (rule) {
        case R_LIN_HALF: return persist_rule<R_LIN_HALF, FQNM_K2P_LIN_V>(a, r, st);
        case R_EO_P1: return persist_rule<R_EO_P1>(a, r, st);
        case R_EO_FAST: return persist_rule<R_EO_FAST>(a, r, st);
        case R_LIN_FAST: return persist_rule<R_LIN_FAST>(a, r, st);
        default: return cudaErrorInvalidValue;
    }
}
#endif

// ---------------------------------------------------------------------------
// K1: naive, one thread per cell, one step per launch
template <int RULE>
__global__ void k_naive(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n,
                        int64_t batch, int bmode, DevRule r)
{
    const int64_t total = n * batch;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / n, i = t - b * n;
        const int32_t* s = src + b * n;
        int64_t il = i - 1, ir = i + 1;
        if (bmode == BM_PERIODIC) {
            if (il < 0) il += n;
            if (ir >= n) ir -= n;
        } else {
            if (il < 0) il = 0;
            if (ir >= n) ir = n - 1;
        }
        if (RULE == R_TWOPOINT || RULE == R_TP_FAST) {
            dst[b * n + i] = s[i] - (tp_eval<RULE>(s[i], s[ir], r) - tp_eval<RULE>(s[il], s[i], r));
            continue;
        }
        int32_t pl, ml, pc, mc, pr, mr;
        phi_pm<RULE>(s[il], pl, ml, r);
        phi_pm<RULE>(s[i], pc, mc, r);
        phi_pm<RULE>(s[ir], pr, mr, r);
        const int32_t Fr = pc + mr, Fl = pl + mc;
        dst[b * n + i] = s[i] - (Fr - Fl);
    }
}

// ---------------------------------------------------------------------------
// K6: resident stepper for one mid-size problem (e.g. BJ.cfg2, N = 65536).
// The domain is split over P warps; warp w owns S_w cells, held with H halo
// cells on each side in a register window of 32*V cells, for ALL nsteps.
// After every block of k <= H steps each warp publishes its H edge cells to
// global memory (double-buffered by block parity: a neighbour can be at most
// one block ahead), raises its flag (release) and waits for both neighbours'
// flags (acquire) before reloading its halos through L2 - no grid-wide
// barrier, no relaunch.  All warps must be co-resident: the launcher uses a
// cooperative launch.  Flags carry tag_base + block, strictly increasing across
// calls, so they never need resetting.
struct ResidentArgs {
    const int32_t* src;
    int32_t* dst;
    int32_t* edges;           // [2 parities][P][2 sides][H]
    unsigned int* flags;      // [P]
    int64_t n;
    int64_t nsteps;
    int32_t P, base, rem, H, k, bmode;   // warp w owns base + (w < rem) cells
    uint32_t tag_base;
};

// launch-bounds minimum of K6: 1 for the two-point Godunov fast path (cfg2 data 166 -> 191
// GCUPS), none for the rest (EO cfg2 371 with none, 358 with 1); -1 = this per-rule choice
#ifndef FQNM_K6_MINB
#define FQNM_K6_MINB -1
#endif
template <int RULE>
constexpr int k6_minb() { return FQNM_K6_MINB >= 0 ? FQNM_K6_MINB : (RULE == R_TP_FAST ? 1 : 0); }

template <int RULE, int V>
__global__ void __launch_bounds__(256, k6_minb<RULE>()) k_resident(ResidentArgs a, DevRule r)
{
    const int lane = threadIdx.x & 31;
    const int w = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (w >= a.P) return;                              // whole warps only
    const int H = a.H;
    const int64_t own0 = (int64_t)w * a.base + (w < a.rem ? w : a.rem);   // first owned cell
    const int Sw = a.base + (w < a.rem ? 1 : 0);
    const int64_t ws = own0 - H;                       // window start (global index)
    const bool wall = a.bmode == BM_TRANSMISSIVE;
    const int wl = (w + a.P - 1) % a.P, wr = (w + 1) % a.P;
    int32_t q[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int pos = lane * V + j;
        int64_t gi = ws + pos;
        if (pos >= H + Sw + H) gi = own0;              // beyond the window's use: any valid state
        if (wall) gi = gi < 0 ? 0 : (gi >= a.n ? a.n - 1 : gi);
        else gi = ((gi % a.n) + a.n) % a.n;
        q[j] = a.src[gi];
    }
    int64_t done = 0;
    uint32_t blk = 0;
    while (done < a.nsteps) {
        const int kb = (int)((a.nsteps - done) < a.k ? (a.nsteps - done) : a.k);
        if (wall)
            run_window_steps<RULE, V, true>(q, kb, r, ws + (int64_t)lane * V, a.n);
        else
            run_window_steps_signed<RULE, V, true>(q, kb, r);
        done += kb;
        if (done >= a.nsteps) break;
        ++blk;
        const uint32_t tag = a.tag_base + blk;
#if FQNM_RES_LL
        // edge exchange in 8-byte {value, tag} words (single-copy atomic): the writer needs
        // no fence and no flag, the reader polls the words it needs until every tag is the
        // block's.  Slot (blk & 1) is safe to overwrite two blocks later: by then the
        // neighbour has read it (its block blk+1 needed these edges).
        {
            uint64_t* e = reinterpret_cast<uint64_t*>(a.edges) + ((size_t)(blk & 1) * a.P + w) * 2 * H;
            const uint64_t hi = (uint64_t)tag << 32;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int pos = lane * V + j;
                if (pos >= H && pos < 2 * H)
                    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(e + pos - H),
                                 "l"(hi | (uint32_t)q[j]) : "memory");
                if (pos >= Sw && pos < Sw + H)
                    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(e + H + pos - Sw),
                                 "l"(hi | (uint32_t)q[j]) : "memory");
            }
            const uint64_t* el = reinterpret_cast<const uint64_t*>(a.edges) +
                                 ((size_t)(blk & 1) * a.P + wl) * 2 * H + H;   // left nbr's right edge
            const uint64_t* er = reinterpret_cast<const uint64_t*>(a.edges) +
                                 ((size_t)(blk & 1) * a.P + wr) * 2 * H;       // right nbr's left edge
            bool need[V];
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int pos = lane * V + j;
                need[j] = pos < H || (pos >= H + Sw && pos < H + Sw + H);
            }
            const long long t0 = clock64();
            for (;;) {
                bool ok = true;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    if (!need[j]) continue;
                    const int pos = lane * V + j;
                    const uint64_t* src = pos < H ? el + pos : er + pos - H - Sw;
                    uint64_t v;
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(src) : "memory");
                    if ((uint32_t)(v >> 32) == tag) {
                        q[j] = (int32_t)(uint32_t)v;
                        need[j] = false;
                    } else {
                        ok = false;
                    }
                }
                if (__all_sync(FULL, ok)) break;
                if (clock64() - t0 > SPIN_TRAP_CYCLES) __trap();
            }
        }
        continue;
#endif
        // publish the edges: left = positions [H, 2H), right = [Sw, Sw + H)
        int32_t* e = a.edges + ((size_t)(blk & 1) * a.P + w) * 2 * H;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int pos = lane * V + j;
            if (pos >= H && pos < 2 * H) e[pos - H] = q[j];
            if (pos >= Sw && pos < Sw + H) e[H + pos - Sw] = q[j];
        }
        __syncwarp();
        if (lane == 0) {
#if FQNM_RES_FENCE == 0
            __threadfence();
#else
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
            asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(a.flags + w), "r"(tag) : "memory");
            unsigned int f;
            const long long t0 = clock64();
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.flags + wl) : "memory");
                if (clock64() - t0 > SPIN_TRAP_CYCLES) __trap();
            } while ((int)(f - tag) < 0);
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.flags + wr) : "memory");
                if (clock64() - t0 > SPIN_TRAP_CYCLES) __trap();
            } while ((int)(f - tag) < 0);
        }
        __syncwarp();
        const int32_t* el = a.edges + ((size_t)(blk & 1) * a.P + wl) * 2 * H + H;   // left nbr's right edge
        const int32_t* er = a.edges + ((size_t)(blk & 1) * a.P + wr) * 2 * H;       // right nbr's left edge
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const int pos = lane * V + j;
            if (pos < H) q[j] = __ldcg(el + pos);
            else if (pos >= H + Sw && pos < H + Sw + H) q[j] = __ldcg(er + pos - H - Sw);
        }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int pos = lane * V + j;
        if (pos >= H && pos < H + Sw) a.dst[ws + pos] = q[j];
    }
}

// ---------------------------------------------------------------------------
// K7: 2D directional composition (Thm formal Cartesian extension):
//   q'_{i,j} = q - (F^x_{i+1/2,j} - F^x_{i-1/2,j}) - (F^y_{i,j+1/2} - F^y_{i,j-1/2})
// A CTA (32 x 16 threads) owns a (TX + 2k) x (TY + 2k) region; every thread keeps
// its fixed cells (x = tx + 32a, y = ty + 16b) in registers for the k steps.
// Per step each thread reads the neighbours' maps (phi+ of the left/lower cell,
// phi- of the right/upper cell) from shared memory, updates its cells, and
// writes the maps of the new values into the other half of a double-buffered
// map array: one barrier per step.  Garbage from the region edge moves in one
// cell per step and the inner TX x TY tile is stored after k steps.
// SAME: identical x and y rules (maps evaluated once).
template <int RULE, bool SAME, bool WALL>
__global__ void __launch_bounds__(512) k_step2d(Step2DArgs a, DevRule rx, DevRule ry)
{
    if (a.guard && *a.guard) return;                    // state left the range earlier
    unsigned gacc = 0;                                  // range guard accumulator (md_acc)
    extern __shared__ int32_t sm2[];
    constexpr int TX = STEP2D_TX, TY = STEP2D_TY;
    constexpr int NA = (TX + 2 * STEP2D_KMAX + 31) / 32;       // cell columns per thread
    constexpr int NB = (TY + 2 * STEP2D_KMAX + 15) / 16;       // cell rows per thread
    const int K = a.ksteps;
    const int RX = TX + 2 * K, RY = TY + 2 * K, R = RX * RY;
    constexpr int NMAP = SAME ? 2 : 4;                          // Px, Mx (, Py, My)
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t nx = a.nx, ny = a.ny;
    const int64_t ox = (int64_t)blockIdx.x * TX - K, oy = (int64_t)blockIdx.y * TY - K;
    int32_t q[NB][NA];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int y = ty + 16 * b;
        int64_t gj = oy + (y < RY ? y : RY - 1);
        if (WALL) gj = gj < 0 ? 0 : (gj >= ny ? ny - 1 : gj);
        else gj = (gj % ny + ny) % ny;
#pragma unroll
        for (int c = 0; c < NA; ++c) {
            const int x = tx + 32 * c;
            int64_t gi = ox + (x < RX ? x : RX - 1);
            if (WALL) gi = gi < 0 ? 0 : (gi >= nx ? nx - 1 : gi);
            else gi = (gi % nx + nx) % nx;
            q[b][c] = a.src[gj * nx + gi];
        }
    }
    // maps of the current values -> buffer 0
    auto publish = [&](int buf) {
        int32_t* M0 = sm2 + (size_t)buf * NMAP * R;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                const int x = tx + 32 * c, y = ty + 16 * b;
                if (x < RX && y < RY) {
                    const int i = y * RX + x;
                    int32_t g, m;
                    phi_gm<RULE>(q[b][c], g, m, rx);
                    M0[i] = g - m;                    // phi+_x
                    M0[R + i] = m;                    // phi-_x
                    if (!SAME) {
                        phi_gm<RULE>(q[b][c], g, m, ry);
                        M0[2 * R + i] = g - m;        // phi+_y
                        M0[3 * R + i] = m;            // phi-_y
                    }
                }
            }
    };
    publish(0);
    __syncthreads();
    for (int s = 0; s < K; ++s) {
        const int32_t* Mc = sm2 + (size_t)(s & 1) * NMAP * R;
        const int32_t* PX = Mc;
        const int32_t* MX = Mc + R;
        const int32_t* PY = SAME ? PX : Mc + 2 * R;
        const int32_t* MY = SAME ? MX : Mc + 3 * R;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                const int x = tx + 32 * c, y = ty + 16 * b;
                if (x < RX && y < RY) {
                    const int i = y * RX + x;
                    const int il = x > 0 ? i - 1 : i, ir = x < RX - 1 ? i + 1 : i;
                    const int id = y > 0 ? i - RX : i, iu = y < RY - 1 ? i + RX : i;
                    int32_t txl = PX[il] + MX[i];
                    int32_t txr = PX[i] + MX[ir];
                    int32_t tyl = PY[id] + MY[i];
                    int32_t tyr = PY[i] + MY[iu];
                    if (WALL) {                                       // ghost copies (A12)
                        const int64_t gi = ox + x, gj = oy + y;
                        if (gi == 0) txl = PX[i] + MX[i];
                        if (gi == nx - 1) txr = PX[i] + MX[i];
                        if (gj == 0) tyl = PY[i] + MY[i];
                        if (gj == ny - 1) tyr = PY[i] + MY[i];
                    }
                    q[b][c] = q[b][c] + txl - txr + tyl - tyr;
                    // range guard on the intermediate steps too (valid cells of the
                    // shrinking trapezoid inside the domain; the last step at the store)
                    if (a.guard && s + 1 < K && x > s && x < RX - 1 - s && y > s && y < RY - 1 - s) {
                        const int64_t gi = ox + x, gj = oy + y;
                        if (gi >= 0 && gi < nx && gj >= 0 && gj < ny) md_acc(gacc, q[b][c], a.glo);
                    }
                }
            }
        if (s + 1 < K) {
            publish((s + 1) & 1);
            __syncthreads();
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < NA; ++c) {
            const int x = tx + 32 * c, y = ty + 16 * b;
            const int64_t gi = ox + x, gj = oy + y;
            if (x >= K && x < K + TX && y >= K && y < K + TY && gi < nx && gj < ny) {
                a.dst[gj * nx + gi] = q[b][c];
                md_acc(gacc, q[b][c], a.glo);
            }
        }
    md_flush(a.guard, gacc, a.glo, a.ghi);
}

#if FQNM_PART(2)
template <int RULE, bool SAME>
static cudaError_t step2d_rule(const Step2DArgs& a, const DevRule& rx, const DevRule& ry,
                               cudaStream_t st)
{
    const int K = a.ksteps;
    const size_t R = (size_t)(STEP2D_TX + 2 * K) * (STEP2D_TY + 2 * K);
    const size_t smem = R * sizeof(int32_t) * 2 * (SAME ? 2 : 4);    // double-buffered maps
    dim3 grid((unsigned)((a.nx + STEP2D_TX - 1) / STEP2D_TX), (unsigned)((a.ny + STEP2D_TY - 1) / STEP2D_TY));
    cudaError_t e;
    if (a.bmode == BM_TRANSMISSIVE) {
        e = cudaFuncSetAttribute(k_step2d<RULE, SAME, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_step2d<RULE, SAME, true><<<grid, 512, smem, st>>>(a, rx, ry);
    } else {
        e = cudaFuncSetAttribute(k_step2d<RULE, SAME, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_step2d<RULE, SAME, false><<<grid, 512, smem, st>>>(a, rx, ry);
    }
    return cudaGetLastError();
}

cudaError_t launch_step2d(int rule, bool same, const Step2DArgs& a, const DevRule& rx,
                          const DevRule& ry, cudaStream_t st)
{
    if (a.ksteps < 1 || a.ksteps > STEP2D_KMAX) return cudaErrorInvalidValue;
    switch (rule) {
        case R_LIN_HALF: return same ? step2d_rule<R_LIN_HALF, true>(a, rx, ry, st)
                                     : step2d_rule<R_LIN_HALF, false>(a, rx, ry, st);
        case R_EO_FAST: return same ? step2d_rule<R_EO_FAST, true>(a, rx, ry, st)
                                    : step2d_rule<R_EO_FAST, false>(a, rx, ry, st);
        case R_EO_P1: return same ? step2d_rule<R_EO_P1, true>(a, rx, ry, st)
                                    : step2d_rule<R_EO_P1, false>(a, rx, ry, st);
        case R_GENERIC: return same ? step2d_rule<R_GENERIC, true>(a, rx, ry, st)
                                    : step2d_rule<R_GENERIC, false>(a, rx, ry, st);
        case R_LIN_FAST: return same ? step2d_rule<R_LIN_FAST, true>(a, rx, ry, st)
                                     : step2d_rule<R_LIN_FAST, false>(a, rx, ry, st);
        default: return cudaErrorInvalidValue;
    }
}

#endif  // part 2

// ---------------------------------------------------------------------------
// K3: one problem of 32*V cells per warp, all steps in registers
#ifndef FQNM_K3_MINB
#define FQNM_K3_MINB 0                    // launch-bounds minimum of K3 (0 = none)
#endif
template <int RULE, int V, bool WALL>
__global__ void __launch_bounds__(128, FQNM_K3_MINB) k_warp_ensemble(int32_t* __restrict__ q, int64_t batch,
                                                        int64_t nsteps, DevRule r)
{
    constexpr int N = 32 * V;
    const int lane = threadIdx.x & 31;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= batch) return;
    int32_t* qb = q + b * N + lane * V;
    int32_t c[V];
    if (V >= 4) {
#pragma unroll
        for (int j = 0; j < V / 4; ++j) {
            int4 v = reinterpret_cast<const int4*>(qb)[j];
            c[4 * j] = v.x; c[4 * j + 1] = v.y; c[4 * j + 2] = v.z; c[4 * j + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j) c[j] = qb[j];
    }
    const int64_t g0 = (int64_t)lane * V;
    int64_t s = 0;
    for (; s + 2 <= nsteps; s += 2) {
        one_step<RULE, V, WALL, 1>(c, r, lane, g0, N);
        one_step<RULE, V, WALL, 1>(c, r, lane, g0, N);
    }
    if (s < nsteps) one_step<RULE, V, WALL, 1>(c, r, lane, g0, N);
    if (V >= 4) {
#pragma unroll
        for (int j = 0; j < V / 4; ++j)
            reinterpret_cast<int4*>(qb)[j] = make_int4(c[4 * j], c[4 * j + 1], c[4 * j + 2],
                                                       c[4 * j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j) qb[j] = c[j];
    }
}

// ---------------------------------------------------------------------------
// K4: one problem per CTA, state and maps in shared memory
template <int RULE>
__global__ void __launch_bounds__(1024) k_cta_ensemble(int32_t* __restrict__ q, int64_t n,
                                                       int64_t nsteps, int bmode, DevRule r)
{
    extern __shared__ int32_t sm[];
    int32_t* Q = sm;
    int32_t* P = sm + n;
    int32_t* M = sm + 2 * n;
    int32_t* qb = q + (int64_t)blockIdx.x * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) Q[i] = qb[i];
    __syncthreads();
    for (int64_t s = 0; s < nsteps; ++s) {
        if constexpr (RULE == R_TWOPOINT || RULE == R_TP_FAST) {
            // P[i] = T_{i+1/2} = Phi(q_i, q_{i+1}) (ghost/wrap as the boundary says)
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                int64_t ir = i + 1;
                if (ir >= n) ir = (bmode == BM_PERIODIC) ? 0 : n - 1;
                P[i] = tp_eval<RULE>(Q[i], Q[ir], r);
            }
            __syncthreads();
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const int32_t Fl = (i > 0) ? P[i - 1]
                                 : (bmode == BM_PERIODIC ? P[n - 1] : tp_eval<RULE>(Q[0], Q[0], r));
                Q[i] = Q[i] - (P[i] - Fl);
            }
            __syncthreads();
        } else {
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) phi_pm<RULE>(Q[i], P[i], M[i], r);
            __syncthreads();
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                int64_t il = i - 1, ir = i + 1;
                int32_t Fl, Fr;
                if (bmode == BM_PERIODIC) {
                    if (il < 0) il += n;
                    if (ir >= n) ir -= n;
                    Fl = P[il] + M[i];
                    Fr = P[i] + M[ir];
                } else {
                    Fl = (i == 0) ? P[0] + M[0] : P[il] + M[i];
                    Fr = (i == n - 1) ? P[i] + M[i] : P[i] + M[ir];
                }
                Q[i] = Q[i] - (Fr - Fl);
            }
            __syncthreads();
        }
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) qb[i] = Q[i];
}

// ---------------------------------------------------------------------------
template <int RULE>
__global__ void k_transfer(const int32_t* __restrict__ q, int32_t* __restrict__ pp,
                           int32_t* __restrict__ pm, int64_t n, DevRule r)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t p, m;
        phi_pm<RULE>(q[i], p, m, r);
        // the stepping kernels' float64 form of the EO magnitude (eo_g_dp) must agree with
        // the float32 + integer-remainder form the hook evaluates: a disagreement poisons
        // the output, so the exhaustive map tests cover both forms
        if (RULE == R_EO_P1 && r.eo_dp_ok && eo_g_dp(q[i], r) != p + m) p = INT32_MIN;
        pp[i] = p;
        pm[i] = m;
    }
}

template <typename T>
__global__ void k_minmax(const T* __restrict__ q, int64_t n, long long* out)
{
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        long long v = (long long)q[i];
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long a = __shfl_xor_sync(FULL, lo, o), b = __shfl_xor_sync(FULL, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, lo);
        atomicMax(out + 1, hi);
    }
}

template <typename T>
__global__ void k_observe(const T* __restrict__ q, double delta, double* __restrict__ u, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        u[i] = __dmul_rn(delta, (double)q[i]);          // u = fl(delta q)
}

// ---------------------------------------------------------------------------
// launchers
static inline int grid_for(int64_t work, int threads, int cap)
{
    int64_t g = (work + threads - 1) / threads;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

template <int RULE, int V, int MINB, int FSIGN = 0>
cudaError_t blocked_v(const BlockedArgs& a, const DevRule& r, cudaStream_t st, int cap)
{
    const int threads = 256;
    int64_t warps = a.nwin * a.batch;
    int g = grid_for(warps * 32, threads, cap);
    k_blocked<RULE, V, MINB, FSIGN><<<g, threads, 0, st>>>(a, r);
    return cudaGetLastError();
}

#ifndef FQNM_BLOCKED_MINB0
#define FQNM_BLOCKED_MINB0 0      // launch-bounds minimum of the uncapped (minb = 0) variants:
                                  // none (exact two-point EO2 132 vs 124 GCUPS with 1, LF 65.6 vs
                                  // 65.1, generic linear 194 vs 195; tools/sweep_generic.py)
#endif
// minb: __launch_bounds__ min blocks per SM (register cap), 0 = default
template <int RULE>
cudaError_t blocked_rule(int V, int minb, const BlockedArgs& a, const DevRule& r,
                                cudaStream_t st, int cap)
{
    if (minb) {
#ifdef FQNM_EXTRA_VARIANTS
        if (V == 32 && minb == 3) return blocked_v<RULE, 32, 3>(a, r, st, cap);
        if (V == 64 && minb == 2) return blocked_v<RULE, 64, 2>(a, r, st, cap);
        if (V == 64 && minb == 1) return blocked_v<RULE, 64, 1>(a, r, st, cap);
        if (V == 48 && minb == 2) return blocked_v<RULE, 48, 2>(a, r, st, cap);
        if (V == 40 && minb == 2) return blocked_v<RULE, 40, 2>(a, r, st, cap);
#endif
        if (V == 16 && minb == 3) return blocked_v<RULE, 16, 3>(a, r, st, cap);
        if (V == 16 && minb == 4) return blocked_v<RULE, 16, 4>(a, r, st, cap);
        if (V == 32 && minb == 2) return blocked_v<RULE, 32, 2>(a, r, st, cap);
        if (V == 8 && minb == 4) return blocked_v<RULE, 8, 4>(a, r, st, cap);
    }
    switch (V) {
        case 8: return blocked_v<RULE, 8, FQNM_BLOCKED_MINB0>(a, r, st, cap);
        case 16: return blocked_v<RULE, 16, FQNM_BLOCKED_MINB0>(a, r, st, cap);
        case 32: return blocked_v<RULE, 32, FQNM_BLOCKED_MINB0>(a, r, st, cap);
        default: return cudaErrorInvalidValue;
    }
}

// per-rule instantiations of the blocked kernels, one translation unit each
#if FQNM_PART(1)
template cudaError_t blocked_rule<R_LIN_HALF>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif
#if FQNM_PART(5)
template cudaError_t blocked_rule<R_EO_FAST>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
template cudaError_t blocked_rule<R_EO_P1>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif
#if FQNM_PART(4)
bool blocked_sign_has_rule(int rule) { return rule == R_EO_P1 || rule == R_EO_FAST; }

// K2S: V = 48, two 256-thread CTAs per SM (128 registers; the sign step keeps no map array)
cudaError_t launch_blocked_sign(int rule, int sign, const BlockedArgs& a, const DevRule& r,
                                cudaStream_t st, int grid_cap)
{
    constexpr int V = BLOCKED_SIGN_V;
    if (rule == R_EO_P1)
        return sign == 1 ? blocked_v<R_EO_P1, V, 2, 1>(a, r, st, grid_cap)
                         : blocked_v<R_EO_P1, V, 2, 2>(a, r, st, grid_cap);
    if (rule == R_EO_FAST)
        return sign == 1 ? blocked_v<R_EO_FAST, V, 2, 1>(a, r, st, grid_cap)
                         : blocked_v<R_EO_FAST, V, 2, 2>(a, r, st, grid_cap);
    return cudaErrorInvalidValue;
}
#endif
#if FQNM_PART(8)
template cudaError_t blocked_v<R_GENERIC, 32, FQNM_BLOCKED_MINB0>(const BlockedArgs&, const DevRule&, cudaStream_t, int);
template cudaError_t blocked_v<R_GENERIC, 32, 2>(const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif
#if FQNM_PART(6)
#if FQNM_SCALAR_PART == 6
extern template cudaError_t blocked_v<R_GENERIC, 32, FQNM_BLOCKED_MINB0>(const BlockedArgs&, const DevRule&, cudaStream_t, int);
extern template cudaError_t blocked_v<R_GENERIC, 32, 2>(const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif
template cudaError_t blocked_rule<R_GENERIC>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif
// two-point rules: V = 8 or 16, no register-cap variants (int64 evaluation)
template <>
cudaError_t blocked_rule<R_TWOPOINT>(int V, int minb, const BlockedArgs& a, const DevRule& r,
                                     cudaStream_t st, int cap);
#if FQNM_PART(9)
template cudaError_t blocked_rule<R_TP_FAST>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
template <>
cudaError_t blocked_rule<R_TWOPOINT>(int V, int minb, const BlockedArgs& a, const DevRule& r,
                                     cudaStream_t st, int cap)
{
    if (minb) return cudaErrorInvalidValue;
    if (V == 8) return blocked_v<R_TWOPOINT, 8, FQNM_BLOCKED_MINB0>(a, r, st, cap);
    if (V == 16) return blocked_v<R_TWOPOINT, 16, FQNM_BLOCKED_MINB0>(a, r, st, cap);
    return cudaErrorInvalidValue;
}
#endif
#if FQNM_PART(7)
template cudaError_t blocked_rule<R_LIN_FAST>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif

#if FQNM_PART(1)
#if FQNM_SCALAR_PART == 1
extern template cudaError_t blocked_rule<R_EO_FAST>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
extern template cudaError_t blocked_rule<R_EO_P1>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
extern template cudaError_t blocked_rule<R_GENERIC>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
extern template cudaError_t blocked_rule<R_LIN_FAST>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
extern template cudaError_t blocked_rule<R_TP_FAST>(int, int, const BlockedArgs&, const DevRule&, cudaStream_t, int);
#endif
#ifdef FQNM_EXTRA_VARIANTS
bool blocked_has_V(int V) { return V == 8 || V == 16 || V == 32 || V == 64 || V == 48 || V == 40; }
#else
bool blocked_has_V(int V) { return V == 8 || V == 16 || V == 32; }
#endif
bool blocked_rule_has_V(int rule, int V) { return rule == R_TWOPOINT ? (V == 8 || V == 16) : blocked_has_V(V); }
int blocked_max_V() { return 32; }

cudaError_t launch_blocked(int rule, int V, int minb, const BlockedArgs& a, const DevRule& r,
                           cudaStream_t st, int grid_cap)
{
    switch (rule) {
        case R_LIN_HALF: return blocked_rule<R_LIN_HALF>(V, minb, a, r, st, grid_cap);
        case R_EO_FAST: return blocked_rule<R_EO_FAST>(V, minb, a, r, st, grid_cap);
        case R_EO_P1: return blocked_rule<R_EO_P1>(V, minb, a, r, st, grid_cap);
        case R_GENERIC: return blocked_rule<R_GENERIC>(V, minb, a, r, st, grid_cap);
        case R_LIN_FAST: return blocked_rule<R_LIN_FAST>(V, minb, a, r, st, grid_cap);
        case R_TWOPOINT: return blocked_rule<R_TWOPOINT>(V, minb, a, r, st, grid_cap);
        case R_TP_FAST: return blocked_rule<R_TP_FAST>(V, minb, a, r, st, grid_cap);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_naive(int rule, const int32_t* src, int32_t* dst, int64_t n, int64_t batch,
                         int bmode, const DevRule& r, cudaStream_t st)
{
    const int threads = 256;
    int g = grid_for(n * batch, threads, 148 * 32);
    switch (rule) {
        case R_LIN_HALF: k_naive<R_LIN_HALF><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        case R_EO_FAST: k_naive<R_EO_FAST><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        case R_EO_P1: k_naive<R_EO_P1><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        case R_GENERIC: k_naive<R_GENERIC><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        case R_LIN_FAST: k_naive<R_LIN_FAST><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        case R_TWOPOINT: k_naive<R_TWOPOINT><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        case R_TP_FAST: k_naive<R_TP_FAST><<<g, threads, 0, st>>>(src, dst, n, batch, bmode, r); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

#endif  // part 1

template <int RULE, int V>
static cudaError_t warp_v(int32_t* q, int64_t batch, int64_t nsteps, int bmode, const DevRule& r,
                          cudaStream_t st)
{
    const int threads = 128;
    int64_t g = (batch * 32 + threads - 1) / threads;
    if (bmode == BM_TRANSMISSIVE)
        k_warp_ensemble<RULE, V, true><<<(unsigned)g, threads, 0, st>>>(q, batch, nsteps, r);
    else
        k_warp_ensemble<RULE, V, false><<<(unsigned)g, threads, 0, st>>>(q, batch, nsteps, r);
    return cudaGetLastError();
}

template <int RULE>
cudaError_t warp_rule(int V, int32_t* q, int64_t batch, int64_t nsteps, int bmode,
                             const DevRule& r, cudaStream_t st)
{
    switch (V) {
        case 1: return warp_v<RULE, 1>(q, batch, nsteps, bmode, r, st);
        case 2: return warp_v<RULE, 2>(q, batch, nsteps, bmode, r, st);
        case 4: return warp_v<RULE, 4>(q, batch, nsteps, bmode, r, st);
        case 8: return warp_v<RULE, 8>(q, batch, nsteps, bmode, r, st);
        case 16: return warp_v<RULE, 16>(q, batch, nsteps, bmode, r, st);
        case 32: return warp_v<RULE, 32>(q, batch, nsteps, bmode, r, st);
        default: return cudaErrorInvalidValue;
    }
}

#if FQNM_PART(3)
template cudaError_t warp_rule<R_LIN_HALF>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
template cudaError_t warp_rule<R_EO_FAST>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
template cudaError_t warp_rule<R_EO_P1>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
template cudaError_t warp_rule<R_LIN_FAST>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
#endif
#if FQNM_PART(10)
template cudaError_t warp_rule<R_TWOPOINT>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
template cudaError_t warp_rule<R_TP_FAST>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
#endif
#if FQNM_PART(4)
template cudaError_t warp_rule<R_GENERIC>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
#endif

#if FQNM_PART(2)
template <int RULE, int V>
static cudaError_t resident_v(const ResidentArgsHost& h, const DevRule& r, cudaStream_t st)
{
    ResidentArgs a;
    a.src = h.src; a.dst = h.dst; a.edges = h.edges; a.flags = h.flags; a.n = h.n;
    a.tag_base = h.tag_base;
    a.nsteps = h.nsteps; a.P = h.P; a.base = h.base; a.rem = h.rem; a.H = h.H; a.k = h.k;
    a.bmode = h.bmode;
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    // up to 4 warps per SM: 128-thread CTAs, one per SM, one warp per sub-partition (the
    // run is latency-bound per warp; two warps on a sub-partition halve its step rate)
    const int threads = h.P <= 4 * sms ? 128 : 256;
    const int blocks = (h.P * 32 + threads - 1) / threads;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<RULE, V>, threads, 0);
    if (e != cudaSuccess) return e;
    if (blocks > per_sm * sms) return cudaErrorCooperativeLaunchTooLarge;
    void* args[] = {&a, const_cast<DevRule*>(&r)};
    return cudaLaunchCooperativeKernel((const void*)k_resident<RULE, V>, blocks, threads, args, 0, st);
}

int resident_capacity_warps(int rule, int V)
{
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e;
    if (V == 8) {
        e = rule == R_LIN_HALF ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_LIN_HALF, 8>, 256, 0)
          : rule == R_EO_FAST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_EO_FAST, 8>, 256, 0)
          : rule == R_EO_P1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_EO_P1, 8>, 256, 0)
          : rule == R_LIN_FAST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_LIN_FAST, 8>, 256, 0)
          : rule == R_TWOPOINT ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_TWOPOINT, 8>, 256, 0)
          : rule == R_TP_FAST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_TP_FAST, 8>, 256, 0)
          : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_GENERIC, 8>, 256, 0);
    } else {
        e = rule == R_LIN_HALF ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_LIN_HALF, 4>, 256, 0)
          : rule == R_EO_FAST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_EO_FAST, 4>, 256, 0)
          : rule == R_EO_P1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_EO_P1, 4>, 256, 0)
          : rule == R_LIN_FAST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_LIN_FAST, 4>, 256, 0)
          : rule == R_TWOPOINT ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_TWOPOINT, 4>, 256, 0)
          : rule == R_TP_FAST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_TP_FAST, 4>, 256, 0)
          : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resident<R_GENERIC, 4>, 256, 0);
    }
    if (e != cudaSuccess) return 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return per_sm * sms * 8;
}

cudaError_t launch_resident(int rule, int V, const ResidentArgsHost& h, const DevRule& r,
                            cudaStream_t st)
{
    if (V != 8 && V != 4) return cudaErrorInvalidValue;
    switch (rule) {
        case R_LIN_HALF: return V == 8 ? resident_v<R_LIN_HALF, 8>(h, r, st) : resident_v<R_LIN_HALF, 4>(h, r, st);
        case R_EO_FAST: return V == 8 ? resident_v<R_EO_FAST, 8>(h, r, st) : resident_v<R_EO_FAST, 4>(h, r, st);
        case R_EO_P1: return V == 8 ? resident_v<R_EO_P1, 8>(h, r, st) : resident_v<R_EO_P1, 4>(h, r, st);
        case R_GENERIC: return V == 8 ? resident_v<R_GENERIC, 8>(h, r, st) : resident_v<R_GENERIC, 4>(h, r, st);
        case R_LIN_FAST: return V == 8 ? resident_v<R_LIN_FAST, 8>(h, r, st) : resident_v<R_LIN_FAST, 4>(h, r, st);
        case R_TWOPOINT: return V == 8 ? resident_v<R_TWOPOINT, 8>(h, r, st) : resident_v<R_TWOPOINT, 4>(h, r, st);
        case R_TP_FAST: return V == 8 ? resident_v<R_TP_FAST, 8>(h, r, st) : resident_v<R_TP_FAST, 4>(h, r, st);
        default: return cudaErrorInvalidValue;
    }
}

#endif  // part 2

#if FQNM_PART(3)
#if FQNM_SCALAR_PART == 3
extern template cudaError_t warp_rule<R_GENERIC>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
extern template cudaError_t warp_rule<R_TWOPOINT>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
extern template cudaError_t warp_rule<R_TP_FAST>(int, int32_t*, int64_t, int64_t, int, const DevRule&, cudaStream_t);
#endif
bool warp_ensemble_has_V(int V) { return V == 1 || V == 2 || V == 4 || V == 8 || V == 16 || V == 32; }

cudaError_t launch_warp_ensemble(int rule, int V, int32_t* q, int64_t batch, int64_t nsteps,
                                 int bmode, const DevRule& r, cudaStream_t st)
{
    switch (rule) {
        case R_LIN_HALF: return warp_rule<R_LIN_HALF>(V, q, batch, nsteps, bmode, r, st);
        case R_EO_FAST: return warp_rule<R_EO_FAST>(V, q, batch, nsteps, bmode, r, st);
        case R_EO_P1: return warp_rule<R_EO_P1>(V, q, batch, nsteps, bmode, r, st);
        case R_GENERIC: return warp_rule<R_GENERIC>(V, q, batch, nsteps, bmode, r, st);
        case R_LIN_FAST: return warp_rule<R_LIN_FAST>(V, q, batch, nsteps, bmode, r, st);
        case R_TWOPOINT: return warp_rule<R_TWOPOINT>(V, q, batch, nsteps, bmode, r, st);
        case R_TP_FAST: return warp_rule<R_TP_FAST>(V, q, batch, nsteps, bmode, r, st);
        default: return cudaErrorInvalidValue;
    }
}

#endif  // part 3

#if FQNM_PART(2)
template <int RULE>
static cudaError_t cta_rule(int32_t* q, int64_t n, int64_t batch, int64_t nsteps, int bmode,
                            const DevRule& r, cudaStream_t st)
{
    size_t smem = (size_t)n * 3 * sizeof(int32_t);
    cudaError_t e = cudaFuncSetAttribute(k_cta_ensemble<RULE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int threads = n >= 1024 ? 1024 : (int)((n + 31) / 32 * 32);
    k_cta_ensemble<RULE><<<(unsigned)batch, threads, smem, st>>>(q, n, nsteps, bmode, r);
    return cudaGetLastError();
}

cudaError_t launch_cta_ensemble(int rule, int32_t* q, int64_t n, int64_t batch, int64_t nsteps,
                                int bmode, const DevRule& r, cudaStream_t st)
{
    switch (rule) {
        case R_LIN_HALF: return cta_rule<R_LIN_HALF>(q, n, batch, nsteps, bmode, r, st);
        case R_EO_FAST: return cta_rule<R_EO_FAST>(q, n, batch, nsteps, bmode, r, st);
        case R_EO_P1: return cta_rule<R_EO_P1>(q, n, batch, nsteps, bmode, r, st);
        case R_GENERIC: return cta_rule<R_GENERIC>(q, n, batch, nsteps, bmode, r, st);
        case R_LIN_FAST: return cta_rule<R_LIN_FAST>(q, n, batch, nsteps, bmode, r, st);
        case R_TWOPOINT: return cta_rule<R_TWOPOINT>(q, n, batch, nsteps, bmode, r, st);
        case R_TP_FAST: return cta_rule<R_TP_FAST>(q, n, batch, nsteps, bmode, r, st);
        default: return cudaErrorInvalidValue;
    }
}

#endif  // part 2

#if FQNM_PART(1)
template <int RULE>
__global__ void k_transfer2(const int32_t* __restrict__ qL, const int32_t* __restrict__ qR,
                            int32_t* __restrict__ T, int64_t n, DevRule r)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        T[i] = transfer_lr<RULE>(qL[i], qR[i], r);
}

cudaError_t launch_transfer2(int rule, const int32_t* qL, const int32_t* qR, int32_t* T, int64_t n,
                             const DevRule& r, cudaStream_t st)
{
    int g = grid_for(n, 256, 148 * 16);
    switch (rule) {
        case R_LIN_HALF: k_transfer2<R_LIN_HALF><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        case R_EO_FAST: k_transfer2<R_EO_FAST><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        case R_EO_P1: k_transfer2<R_EO_P1><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        case R_GENERIC: k_transfer2<R_GENERIC><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        case R_LIN_FAST: k_transfer2<R_LIN_FAST><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        case R_TWOPOINT: k_transfer2<R_TWOPOINT><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        case R_TP_FAST: k_transfer2<R_TP_FAST><<<g, 256, 0, st>>>(qL, qR, T, n, r); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_transfer(int rule, const int32_t* q, int32_t* pp, int32_t* pm, int64_t n,
                            const DevRule& r, cudaStream_t st)
{
    int g = grid_for(n, 256, 148 * 16);
    switch (rule) {
        case R_LIN_HALF: k_transfer<R_LIN_HALF><<<g, 256, 0, st>>>(q, pp, pm, n, r); break;
        case R_EO_FAST: k_transfer<R_EO_FAST><<<g, 256, 0, st>>>(q, pp, pm, n, r); break;
        case R_EO_P1: k_transfer<R_EO_P1><<<g, 256, 0, st>>>(q, pp, pm, n, r); break;
        case R_GENERIC: k_transfer<R_GENERIC><<<g, 256, 0, st>>>(q, pp, pm, n, r); break;
        case R_LIN_FAST: k_transfer<R_LIN_FAST><<<g, 256, 0, st>>>(q, pp, pm, n, r); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

__global__ void k_range_guard(const int32_t* __restrict__ q, int64_t n, long long lo, long long hi,
                              int* flag)
{
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const long long v = q[i];
        bad |= (v < lo) | (v > hi);
    }
    if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void k_range_sign_guard(const int32_t* __restrict__ q, int64_t n, long long lo,
                                   long long hi, int* flag, int* sign_bits)
{
    bool bad = false, neg = false, pos = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const long long v = q[i];
        bad |= (v < lo) | (v > hi);
        neg |= v < 0;
        pos |= v > 0;
    }
    const bool b = __any_sync(FULL, bad), ng = __any_sync(FULL, neg), ps = __any_sync(FULL, pos);
    if ((threadIdx.x & 31) == 0) {
        if (b) atomicOr(flag, 1);
        if (ng || ps) atomicOr(sign_bits, (ng ? 1 : 0) | (ps ? 2 : 0));
    }
}

cudaError_t launch_range_sign_guard(const int32_t* q, int64_t n, long long lo, long long hi,
                                    int* flag, int* sign_bits, cudaStream_t st)
{
    k_range_sign_guard<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(q, n, lo, hi, flag, sign_bits);
    return cudaGetLastError();
}

cudaError_t launch_range_guard(const int32_t* q, int64_t n, long long lo, long long hi, int* flag,
                               cudaStream_t st)
{
    k_range_guard<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(q, n, lo, hi, flag);
    return cudaGetLastError();
}

cudaError_t launch_minmax(const void* q, int dtype, int64_t n, long long* out2, cudaStream_t st)
{
    int g = grid_for(n, 256, 148 * 8);
    if (dtype == 0)
        k_minmax<int32_t><<<g, 256, 0, st>>>((const int32_t*)q, n, out2);
    else
        k_minmax<int64_t><<<g, 256, 0, st>>>((const int64_t*)q, n, out2);
    return cudaGetLastError();
}

cudaError_t launch_observe(const void* q, int dtype, double delta, double* u, int64_t n,
                           cudaStream_t st)
{
    int g = grid_for(n, 256, 148 * 16);
    if (dtype == 0)
        k_observe<int32_t><<<g, 256, 0, st>>>((const int32_t*)q, delta, u, n);
    else
        k_observe<int64_t><<<g, 256, 0, st>>>((const int64_t*)q, delta, u, n);
    return cudaGetLastError();
}

#endif  // part 1

}  // namespace fqnm
