// Internal declarations shared by the host planner (fqnm_api.cu) and the kernels.
// Not part of the C ABI (include/fqnm.h is).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fqnm {

// ---- device rule: how the kernels evaluate (phi+, phi-) ------------------
// Selected by the planner (rule builder) from the exact rational maps.
enum RuleKind : int32_t {
    R_LIN_HALF = 1,   // LINEAR a > 0, kappa = 1/2 exactly, RHA: phi+ = q - trunc(q/2), phi- = 0
    R_EO_FAST = 2,    // BURGERS_EO, RHA: g(|q|) = floor((2P q^2 + Q)/(2Q)) by float estimate +
                      // exact 32-bit remainder correction (valid range proven at plan time)
    R_GENERIC = 3,    // any piecewise-quadratic map, exact int64 arithmetic, any rounding
    R_EO_P1 = 5,      // BURGERS_EO with P = 1 (kappa = 1/Q): as R_EO_FAST, remainder in the
                      // (q^2 - Q est) form, one instruction shorter (maps.cuh eo_gm_p1)
    R_TWOPOINT = 6,   // quantised two-point rule Phi(qL, qR) rounded once (Godunov / EO2 / LF2),
                      // exact int64 evaluation (maps.cuh tp_phi)
    R_TP_FAST = 7,    // two-point Godunov on the EO closed-form domain: Phi = g(max(qL+, -qR-))
                      // with the EO magnitude g (maps.cuh tp_godunov_fast)
    R_LIN_FAST = 4    // LINEAR any |kappa| <= 1, RHA: g(|q|) = floor((2P|q| + Q)/(2Q)) by the
                      // same estimate + remainder scheme as EO (eo_* constants), sign restored
};

enum Support : int32_t { SUPP_ALL = 0, SUPP_POS = 1, SUPP_NEG = 2, SUPP_NONE = 3 };

struct DevRule {
    // generic maps: phi(q) = [q in supp] round((c2 q^2 + c1 q)/den)
    int64_t c2p, c1p, denp;
    int64_t c2m, c1m, denm;
    int32_t suppp, suppm;
    int32_t rounding;
    // EO fast path constants (maps.cuh eo_g)
    int32_t eo_ntwoP;     // -2P
    int32_t eo_c1;        // Q - 1 - 2Q * 0x4B400000  (mod 2^32)
    int32_t eo_twoQ;      // 2Q
    float eo_cf;          // largest float <= (P/Q)(1 - 2^-21)
    int32_t lin_minus;    // R_LIN_FAST: 0 -> the map is phi+ (a > 0), 1 -> phi- (a < 0)
    int32_t one;          // runtime 1 and -1: let the linear kernel issue IMADs (FMA pipe)
    int32_t mone;
    // EO remainder in the (P q^2 - Q est) form (maps.cuh eo_gm_p1, P = 1)
    int32_t eo_nQ;        // -Q
    int32_t eo_c6;        // Q * 0x4B400001 - ceil(Q/2)  (mod 2^32)
    int32_t eo_P;         // P
    // EO magnitude map in float64 (maps.cuh eo_g_dp): g = rint((q^2) * eo_dinv) exactly
    int32_t eo_dp_ok;     // planner: P q^2 < 2^44 on the admissible range
    long long eo_xoff;    // bits of 2^52 (ulp 1): X = q*q + eo_xoff is the double 2^52 + q^2
    double eo_dinv;       // (P/Q)(1 + 2^-46), rounded to double
    double eo_dc1;        // -2^52 * eo_dinv (exact)
    // two-point rule (R_TWOPOINT): Phi = round(num / tp_den),
    //   Godunov: num = c2 max(max(qL,0)^2, min(qR,0)^2); EO2: c2 (max(qL,0)^2 + min(qR,0)^2);
    //   LF2: c2 (qL^2 + qR^2) + c1 (qL - qR)
    int32_t tp_kind;      // 0 = split rule, 5 Godunov, 6 EO2, 7 LF2 (fqnm_flux_kind codes)
    int32_t tp_fast;      // Godunov on the EO fast domain: 1 = EO P = 1 closed form, 2 = general P
    int64_t tp_c2, tp_c1, tp_den;
    // round(num / den) in float64 (maps.cuh round_div_dp; RHA only, |num| < 2^44 on the range):
    // index 0: phi+ (denp), 1: phi- (denm), 2: the two-point rule (tp_den)
    int32_t dv_ok[3];
    double dv_inv[3];     // (1/den)(1 + 2^-46), last two significand bits 0
    double dv_c[3];       // -1.5 2^52 * dv_inv (exact)
};

enum Bmode : int32_t { BM_PERIODIC = 0, BM_TRANSMISSIVE = 1, BM_HALO = 2 };

struct BlockedArgs {
    const int32_t* src;
    int32_t* dst;
    int64_t n;          // cells per problem (owned cells for HALO)
    int64_t batch;
    int64_t nwin;       // windows per problem
    int64_t halo;       // HALO: halo cells each side in src/dst
    int32_t ksteps;
    int32_t KL, KR;     // garbage-shrink per side (multiples of 4)
    int32_t bmode;
    // fused peer-memory halo exchange (HALO plans with p2p): window 0 and the last
    // window push their H edge cells straight into the neighbours' next buffers
    // over NVLink and release a tag; the windows that read halos acquire it first
    int32_t p2p;
    uint32_t tag;                  // tag this block's halos carry / this block pushes + 1
    int32_t* peer_left_dst;        // left neighbour's next ext buffer
    int32_t* peer_right_dst;       // right neighbour's next ext buffer
    int64_t left_n, right_n;       // neighbours' owned cells
    unsigned int* self_flags;      // [0]: left-halo tag, [1]: right-halo tag (written by peers)
    unsigned int* peer_left_flags;
    unsigned int* peer_right_flags;
    const int* guard;              // optional: nonzero -> the launch does nothing (failed range check)
    // dual launch (the sign of the state is only known on the device): bit 0 of *sign_bits
    // set = some cell < 0.  The sign-specialised kernel (K2S) returns when it is set, the
    // general K2 when it is clear.  nullptr: one kernel, chosen by the host.
    const int* sign_bits;
};

struct EulerArgs {
    const int64_t* src;
    int64_t* dst;
    int64_t n;
    int64_t batch;
    int64_t nwin;
    double delta, s, g1;
    double lam;         // dt/dx (density-only variant: float update of m and E)
    int32_t bmode;
    int32_t mode;       // 0: all components quanta, 1: density-only quantisation
};

struct ResidentArgsHost {
    const int32_t* src;
    int32_t* dst;
    int32_t* edges;              // halo edges [2][P][2][H]
    unsigned int* flags;         // [P] block tags
    int64_t n, nsteps;
    int32_t P, base, rem, H, k, bmode;
    uint32_t tag_base;           // tags strictly increase across calls of one plan
};

int resident_capacity_warps(int rule, int V);   // 0 if unavailable (no GPU)

// K7: 2D directional composition, smem-tiled with k <= STEP2D_KMAX steps per launch
#define STEP2D_TX 128
#define STEP2D_TY 32
#define STEP2D_KMAX 4
struct Step2DArgs {
    const int32_t* src;
    int32_t* dst;
    int64_t nx, ny;
    int32_t ksteps;
    int32_t bmode;
    // optional range guard (2D/3D): *guard != 0 -> the launch does nothing;
    // a stored cell outside [glo, ghi] sets *guard
    int* guard;
    int32_t glo, ghi;
};
cudaError_t launch_step2d(int rule, bool same, const Step2DArgs& a, const DevRule& rx,
                          const DevRule& ry, cudaStream_t st);
// K9: 2D streaming, one step per launch, warp per (x strip, y chunk) (kernels_2d.cu);
// a.ksteps carries the rows per chunk
cudaError_t launch_step2d_stream(int rule, bool same, const Step2DArgs& a, const DevRule& rx,
                                 const DevRule& ry, cudaStream_t st);
int64_t step2d_stream_rows(int64_t nx, int64_t ny);
cudaError_t launch_step2d_stream2(int rule, bool same, const Step2DArgs& a, const DevRule& rx,
                                  const DevRule& ry, cudaStream_t st);   // two steps per launch

// K8: 3D directional composition, one step per launch, 2.5D z-streaming (kernels_3d.cu)
struct Step3DArgs {
    const int32_t* src;
    int32_t* dst;
    int64_t nx, ny, nz;
    int64_t zchunk;     // z planes per CTA
    int32_t bmode;
    int32_t xt0;        // first x tile of the launch (set by launch_step3d)
    int* guard;         // optional range guard, as Step2DArgs
    int32_t glo, ghi;
};
cudaError_t launch_step3d(int rule, bool same, const Step3DArgs& a, const DevRule& rx,
                          const DevRule& ry, const DevRule& rz, cudaStream_t st);
int64_t step3d_zchunk(int64_t nx, int64_t ny, int64_t nz);     // z planes per CTA
// K10: 3D warp streaming (two rows of a 124-wide x strip per warp, no inter-warp
// exchange; kernels_3d_s.cu)
cudaError_t launch_step3d_stream(int rule, bool same, const Step3DArgs& a, const DevRule& rx,
                                 const DevRule& ry, const DevRule& rz, cudaStream_t st);
int64_t step3d_s_zchunk(int64_t nx, int64_t ny, int64_t nz);

// level-space diagnostics (kernels_diag.cu)
cudaError_t launch_histogram(const void* q, int dtype, int64_t n, int64_t lo, int64_t L,
                             unsigned int* counts, unsigned long long* outside, cudaStream_t st);
cudaError_t launch_clogc(const unsigned int* counts, int64_t L, double* acc,
                         unsigned long long* occupied, cudaStream_t st);
cudaError_t launch_pairs(const void* q0, const void* q1, int dtype, int64_t n, int64_t lo, int64_t L,
                         unsigned long long* keys, unsigned int* vals, unsigned long long cap,
                         unsigned long long* overflow, cudaStream_t st);
cudaError_t launch_rowsums(const unsigned long long* keys, const unsigned int* vals,
                           unsigned long long cap, int64_t L, const unsigned int* c0, double* rowsum,
                           unsigned long long* npairs, cudaStream_t st);
cudaError_t launch_defect(const double* rowsum, const unsigned int* c0, const unsigned int* c1,
                          int64_t L, unsigned long long* maxbits, cudaStream_t st);

// kernel launchers (kernels_scalar.cu / kernels_euler.cu); return cudaError_t
cudaError_t launch_blocked(int rule, int V, int minb, const BlockedArgs& a, const DevRule& r,
                           cudaStream_t st, int grid_cap);
// K2S: K2 for a state whose cells are all >= 0 (sign 1) or all <= 0 (sign 2), EO rules only,
// V = BLOCKED_SIGN_V cells per lane (no vote, no general path: 128 registers hold V = 48)
#define BLOCKED_SIGN_V 48
bool blocked_sign_has_rule(int rule);
cudaError_t launch_blocked_sign(int rule, int sign, const BlockedArgs& a, const DevRule& r,
                                cudaStream_t st, int grid_cap);
// flag |= 1 if any q[i] outside [lo, hi]; sign_bits |= 1 if any q[i] < 0, 2 if any > 0
cudaError_t launch_range_sign_guard(const int32_t* q, int64_t n, long long lo, long long hi,
                                    int* flag, int* sign_bits, cudaStream_t st);
cudaError_t launch_resident(int rule, int V, const ResidentArgsHost& h, const DevRule& r,
                            cudaStream_t st);

// K2P: persistent temporally blocked stepper (kernels_scalar.cu): all blocks of k steps in
// one launch; warps claim (block, window) items in order from a counter, and an item of
// block b waits (acquire) for the block b-1 items covering its input window (release flags)
struct PersistArgs {
    int32_t* buf0;              // block b reads buf[b & 1], writes buf[(b + 1) & 1]
    int32_t* buf1;
    int64_t n, nwin;
    int32_t S, KL, KR, base, rem, nblocks, bmode, pad;   // block b: base + (b < rem) steps
    unsigned int* flags;        // [nwin]: tag_base + (blocks completed) for the window
    unsigned long long* counter;
    uint32_t tag_base;
    const int* guard;           // the launch returns at once when *guard != 0 (input out of range)
    const int* sign_bits;       // dual launch (pipelined chunks): bit 0 = the input has a negative
                                // cell; the sign-specialised kernel runs when clear, the voting
                                // kernel when set
};
cudaError_t launch_blocked_persist(int rule, int sign, const PersistArgs& a, const DevRule& r,
                                   cudaStream_t st);
bool blocked_persist_has_rule(int rule);
int blocked_persist_V(int rule, int sign);   // cells per lane of the persistent kernel
cudaError_t launch_halo_prime(const BlockedArgs& a, cudaStream_t st);
cudaError_t launch_naive(int rule, const int32_t* src, int32_t* dst, int64_t n, int64_t batch,
                         int bmode, const DevRule& r, cudaStream_t st);
cudaError_t launch_warp_ensemble(int rule, int V, int32_t* q, int64_t batch, int64_t nsteps,
                                 int bmode, const DevRule& r, cudaStream_t st);
cudaError_t launch_cta_ensemble(int rule, int32_t* q, int64_t n, int64_t batch, int64_t nsteps,
                                int bmode, const DevRule& r, cudaStream_t st);
cudaError_t launch_transfer2(int rule, const int32_t* qL, const int32_t* qR, int32_t* T, int64_t n,
                             const DevRule& r, cudaStream_t st);
// transfer-operator equivalence checker (kernels_diag.cu): one step of rule a with
// rule b evaluated on every interface; counters: [0] mismatches, [1] first step (min),
// [2] table overflow
cudaError_t launch_equiv_step(const int32_t* q, int32_t* qn, int32_t* T, int64_t n, int bmode,
                              const DevRule& ra, int rule_a, const DevRule& rb, int rule_b,
                              int64_t step, unsigned long long* counters, unsigned long long* keys,
                              unsigned int* vals, unsigned long long mask, int64_t lo, int64_t L,
                              cudaStream_t st);
cudaError_t launch_equiv_count(const unsigned long long* keys, const unsigned int* vals,
                               unsigned long long cap, unsigned long long* out2, cudaStream_t st);
cudaError_t launch_transfer(int rule, const int32_t* q, int32_t* pp, int32_t* pm, int64_t n,
                            const DevRule& r, cudaStream_t st);
cudaError_t launch_minmax(const void* q, int dtype, int64_t n, long long* out2, cudaStream_t st);
// flag |= any q[i] outside [lo, hi]  (int32 state; asynchronous range check of the e2e pipeline)
cudaError_t launch_range_guard(const int32_t* q, int64_t n, long long lo, long long hi, int* flag,
                               cudaStream_t st);
cudaError_t launch_observe(const void* q, int dtype, double delta, double* u, int64_t n,
                           cudaStream_t st);
cudaError_t launch_euler(int V, const EulerArgs& a, cudaStream_t st);
cudaError_t launch_roe_transfer(const int64_t* qL, const int64_t* qR, int64_t* T, int64_t n,
                                double delta, double s, double g1, cudaStream_t st);

cudaError_t launch_rcp_sqrt_check(int64_t n, uint64_t seed, int e_lo, int e_hi,
                                  unsigned long long* counts, cudaStream_t st);

int blocked_max_V();
bool blocked_has_V(int V);
bool blocked_rule_has_V(int rule, int V);
bool warp_ensemble_has_V(int V);
bool euler_has_V(int V);

}  // namespace fqnm
