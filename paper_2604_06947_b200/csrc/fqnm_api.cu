// Host side of libfqnm: the C ABI of include/fqnm.h, the transfer-rule builder
// (exact kappa, D8 validation, range/headroom, fast-path selection) and the
// planner that picks a kernel family, V and k and drives the launches.
//
// Paper references: Eq. flux_table P:62-68 (maps), Eq. count flux
// P:91-94, update P:86-89, reconstruction P:101-105, CFL/monotonicity Lemma
// P:189-238 (the integer form D8 is checked here), Roe system P:564-575.
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fqnm.h"
#include "fqnm_internal.h"

using namespace fqnm;

typedef __int128 i128;

// ---------------------------------------------------------------------------
// errors
static thread_local std::string g_err;

static int fail(int status, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return status;
}

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(FQNM_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));      \
    } while (0)

// ---------------------------------------------------------------------------
// exact host maps: phi(q) = [q in supp] round((c2 q^2 + c1 q)/den)
struct HostMap {
    int64_t c2 = 0, c1 = 0, den = 1;
    int32_t supp = SUPP_NONE;
};

static i128 floor_div128(i128 num, i128 den)
{
    i128 q = num / den;
    if ((num % den != 0) && (num < 0)) q -= 1;
    return q;
}

static i128 round128(i128 num, i128 den, int rounding)
{
    if (rounding == FQNM_ROUND_FLOOR) return floor_div128(num, den);
    i128 a = num < 0 ? -num : num;
    i128 r;
    if (rounding == FQNM_ROUND_HALF_AWAY) {
        r = (2 * a + den) / (2 * den);
    } else {
        i128 fl = a / den, rem = a - fl * den;
        if (2 * rem > den) r = fl + 1;
        else if (2 * rem < den) r = fl;
        else r = (fl % 2 == 0) ? fl : fl + 1;
    }
    return num < 0 ? -r : r;
}

static int64_t host_phi(const HostMap& m, int64_t q, int rounding)
{
    if (m.supp == SUPP_NONE) return 0;
    if (m.supp == SUPP_POS && q <= 0) return 0;
    if (m.supp == SUPP_NEG && q >= 0) return 0;
    i128 num = (i128)m.c2 * q * q + (i128)m.c1 * q;
    return (int64_t)round128(num, m.den, rounding);
}

static bool map_is_zero(const HostMap& m) { return m.supp == SUPP_NONE || (m.c2 == 0 && m.c1 == 0); }

static int64_t gcd64(int64_t a, int64_t b)
{
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}

// exact rational nearest a positive or negative double: simplest convergent of
// the exact continued fraction of x with den <= 2^31 and |x - p/q| <= 2^-50 |x|
// (a double product of the config's decimals is within 2^-52 of the exact rational)
static bool rationalize(double x, int64_t* pnum, int64_t* pden)
{
    if (!std::isfinite(x) || x == 0.0) return false;
    const bool neg = x < 0;
    double ax = neg ? -x : x;
    int e2;
    double fr = std::frexp(ax, &e2);                  // ax = fr * 2^e2, fr in [0.5, 1)
    int64_t M = (int64_t)std::ldexp(fr, 53);          // exact 53-bit mantissa
    int sh = 53 - e2;                                  // ax = M / 2^sh
    i128 num, den;
    if (sh <= 0) {
        if (-sh > 60) return false;
        num = (i128)M << (-sh);
        den = 1;
    } else {
        if (sh > 120) return false;
        num = M;
        den = (i128)1 << sh;
    }
    // continued fraction of num/den with convergents h/k
    i128 h0 = 0, h1 = 1, k0 = 1, k1 = 0;
    i128 a = num, b = den;
    for (int it = 0; it < 200 && b != 0; ++it) {
        i128 t = a / b;
        i128 h2 = t * h1 + h0, k2 = t * k1 + k0;
        if (k2 > ((i128)1 << 31)) break;
        h0 = h1; h1 = h2; k0 = k1; k1 = k2;
        i128 r = a - t * b;
        a = b; b = r;
        // |num/den - h1/k1| <= 2^-50 num/den  <=>  |num k1 - h1 den| 2^50 <= num k1
        i128 diff = num * k1 - h1 * den;
        if (diff < 0) diff = -diff;
        if (diff <= ((num * k1) >> 50)) {
            if (h1 > INT64_MAX || k1 > INT64_MAX) return false;
            *pnum = neg ? -(int64_t)h1 : (int64_t)h1;
            *pden = (int64_t)k1;
            return true;
        }
    }
    return false;
}

// ---------------------------------------------------------------------------
struct fqnm_plan {
    fqnm_plan_desc d{};
    // rule
    HostMap hp, hm;
    DevRule dr{};
    int rule = 0;
    int64_t kap_num = 0, kap_den = 0;
    int64_t lo = 0, hi = 0;
    bool dep_left = false, dep_right = false;
    // kernel choice
    int family = 0;
    int V = 0;
    int k = 0;
    int minb = 0;         // K2 register cap variant (0 = default)
    // EO plans whose derived D8 range exceeds the fast closed form's domain: [lo, hi] is the
    // fast domain and d8_lim the largest |q| D8 admits; a range-checked step whose state
    // leaves [lo, hi] but stays within +-d8_lim runs on the exact int64 rule (child plan)
    int64_t d8_lim = 0;
    fqnm_plan_t* generic_child = nullptr;
    bool trusted_range = false;         // declared range already D8-validated by the parent
    // Euler constants
    double s_e = 0, g1_e = 0;
    // memory
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    long long* d_minmax = nullptr;
    long long* h_minmax = nullptr;
    void* e2e_dev = nullptr;
    size_t e2e_bytes = 0;
    int32_t* edges = nullptr;           // K6 resident stepper: halo edges + block-tag flags
    unsigned int* flags = nullptr;
    int res_P = 0;
    uint32_t tag_base = 0;
    // fused peer-memory halo exchange (HALO + p2p)
    void* hbuf[2] = {nullptr, nullptr};
    unsigned int* hflags = nullptr;
    int hcur = 0;
    bool hconnected = false;
    void* lbuf[2] = {nullptr, nullptr};
    void* rbuf[2] = {nullptr, nullptr};
    unsigned int* lflags = nullptr;
    unsigned int* rflags = nullptr;
    int64_t ln = 0, rn = 0;
    uint32_t htag = 1;
    // 2D plans (family 7): y-direction rule
    int64_t nx = 0, ny = 0;
    HostMap hpy, hmy;
    DevRule dry{};
    bool same_xy = false;
    bool stream2d = true;               // 2D: K9 streaming instead of K7
    int k2s = 2;                        // K9 steps per launch (1 or 2)
    bool stream3d = false;              // 3D: K10 warp streaming instead of K8 (measured slower)
    // K2P persistent stepper (one launch for all blocks): -1 auto (use_persist: few waves
    // of windows per launch), 0 off (kernel override 2), 1 forced (kernel override 12)
    int persist = -1;
    unsigned int* pflags = nullptr;
    unsigned long long* pcounter = nullptr;
    int64_t pflags_n = 0;
    uint32_t ptag = 1;
    // 3D plans (family 8): z-direction rule
    int64_t nz = 0;
    DevRule drz{};
    cudaStream_t st = nullptr;
    int64_t launches = 0;
    // pipelined end-to-end stepping (fqnm_step_host): chunk plan + 3 ext buffers + streams
    const int* guard = nullptr;          // K2 launches return at once when *guard != 0
    // K2S (sign-specialised K2, EO rules): sign_hint = 1 / 2 when this fqnm_step call's
    // range check proved every cell >= 0 / <= 0 (the maximum principle keeps it for the
    // call); sign_dev = device sign bits of the input (pipelined chunks: dual launch)
    int sign_hint = 0;
    int64_t k2s_launches = 0;            // K2S launches since creation (fqnm_plan_info)
    bool no_sign = false;                // kernel override 2 / 12 / 100m + 2: the general K2 only
    const int* sign_dev = nullptr;
    int* pipe_sign = nullptr;            // per chunk sign bits (pipelined fqnm_step_host)
    int* pipe_sign_host = nullptr;
    int sign_preset = 0;                 // sign_hint a caller (the pipeline) proved for one call
    fqnm_plan_t* pipe_child = nullptr;   // the child plan of the full chunk size C
    int64_t pipe_H = 0, pipe_C = 0, pipe_m = 0;
    // chunk list (ramped: the first and last full chunks are cut into C/8, C/8, C/4, C/2 so the
    // un-overlapped first H2D and last D2H are small); pipe_kids[i] steps chunks of size C >> i
    std::vector<int64_t> pipe_start, pipe_size;
    fqnm_plan_t* pipe_kids[4] = {nullptr, nullptr, nullptr, nullptr};
    void* pipe_buf[3] = {nullptr, nullptr, nullptr};
    int32_t* pipe_head = nullptr;        // copy of q_host[0, H) taken before any D2H (the last
                                         // chunk's periodic right halo)
    int* md_guard = nullptr;             // 2D/3D: state left [lo, hi] during a call (device)
    int* md_guard_host = nullptr;
    int* pipe_guard = nullptr;           // one flag per chunk
    int* pipe_guard_host = nullptr;
    int64_t pipe_guard_n = 0;
    cudaStream_t pipe_h2d = nullptr, pipe_d2h = nullptr;
    // ensemble e2e pipeline (fqnm_step_host on a batched plan): own streams + one event pair per chunk
    cudaStream_t ens_h2d = nullptr, ens_d2h = nullptr;
    cudaEvent_t ens_ev[2 * 16 + 1] = {};
    cudaEvent_t pipe_ev[9] = {};         // [0..2] h2d done, [3..5] compute done, [6..8] d2h done
    // profiling (fqnm_profile_enable)
    bool prof = false;
    std::vector<cudaEvent_t> ev;      // pairs (start, stop)
    size_t ev_used = 0;
};

extern "C" int fqnm_debug_rcp_sqrt(int64_t n, uint64_t seed, int32_t e_lo, int32_t e_hi,
                                   int64_t* mismatches)
{
    if (!mismatches) return fail(FQNM_ERR_ARG, "null argument");
    if (n < 0 || e_lo < -1022 || e_hi > 1023 || e_lo > e_hi)
        return fail(FQNM_ERR_ARG, "exponent range must satisfy -1022 <= e_lo <= e_hi <= 1023");
    unsigned long long* d = nullptr;
    unsigned long long h[4] = {0, 0, 0, 0};
    CUDA_TRY(cudaMalloc(&d, sizeof h));
    cudaError_t e = cudaMemset(d, 0, sizeof h);
    if (e == cudaSuccess && n > 0) e = launch_rcp_sqrt_check(n, seed, e_lo, e_hi, d, 0);
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(FQNM_ERR_CUDA, "rcp/sqrt check: %s", cudaGetErrorString(e));
    for (int i = 0; i < 4; ++i) mismatches[i] = (int64_t)h[i];
    return FQNM_OK;
}

static void fill_info(const fqnm_plan_t* p, fqnm_plan_info* info);
static int plan_build(fqnm_plan_t** out, const fqnm_plan_desc* din, bool allocate,
                      bool trusted_range = false);

// K6 geometry: V = 8 (W = 256 cells per warp), H = round4(k) halo cells per side,
// at most 1184 warps (one 256-thread CTA per SM: always co-resident)
static const int RESIDENT_MAX_WARPS = 148 * 8;
static const int64_t RESIDENT_MAX_CELLS = (int64_t)RESIDENT_MAX_WARPS * (256 - 2 * 16);

static size_t elem_size(const fqnm_plan_desc& d) { return d.dtype == FQNM_I64 ? 8 : 4; }

static size_t state_elems(const fqnm_plan_desc& d)
{
    int64_t n = d.n_local + (d.boundary == FQNM_HALO ? 2 * d.halo : 0);
    return (size_t)d.batch * (size_t)d.nvar * (size_t)n;
}

extern "C" void fqnm_desc_init(fqnm_plan_desc* d)
{
    if (!d) return;
    std::memset(d, 0, sizeof *d);
    d->batch = 1;
    d->nvar = 1;
    d->dtype = FQNM_I32;
    d->rounding = FQNM_ROUND_HALF_AWAY;
    d->boundary = FQNM_PERIODIC;
    d->check_range = 0;
}

// D8 on [lo, hi]: phi+ nondecreasing, phi- nonincreasing, dphi+ - dphi- <= 1.
// Returns the first failing q (lo - 1 if none).
static int64_t d8_first_violation(const fqnm_plan_t* p, int64_t lo, int64_t hi)
{
    int rd = p->d.rounding;
    int64_t pp = host_phi(p->hp, lo, rd), pm = host_phi(p->hm, lo, rd);
    for (int64_t q = lo; q < hi; ++q) {
        int64_t np_ = host_phi(p->hp, q + 1, rd), nm = host_phi(p->hm, q + 1, rd);
        int64_t dp = np_ - pp, dm = nm - pm;
        if (dp < 0 || dm > 0 || dp - dm > 1) return q;
        pp = np_; pm = nm;
    }
    return lo - 1;
}

// headroom of the int64 generic device path: |2 (c2 q^2 + c1 q)| + den < 2^62
static bool generic_headroom(const HostMap& m, int64_t a)
{
    if (map_is_zero(m)) return true;
    i128 A = a;
    i128 num = (i128)(m.c2 < 0 ? -m.c2 : m.c2) * A * A + (i128)(m.c1 < 0 ? -m.c1 : m.c1) * A;
    return 2 * num + m.den < ((i128)1 << 62);
}

// Largest A such that D8 holds on [-A, A] (and the int64 generic path has headroom, and
// A fits the int32 state); 0 if D8 fails already at |q| <= 1.
// EO (c1 = 0, both maps |phi| = round(kappa q^2) on their half-lines): the increment
// round(kappa (a+1)^2) - round(kappa a^2) of a monotone rounding is <= 1 whenever
// kappa (2a + 1) < 1, so the scan starts at a0 = max{a : P (2a + 1) < Q} and only the part
// beyond it (where increments of 2 first appear within ~1/(kappa(2a+1) - 1) steps) is walked.
static int64_t d8_symmetric_limit(const fqnm_plan_t* p, bool eo)
{
    const int rd = p->d.rounding;
    const int64_t cap = INT32_MAX - 1;
    auto room = [&](int64_t a) { return generic_headroom(p->hp, a) && generic_headroom(p->hm, a); };
    int64_t A = 0;
    if (eo) {
        const i128 P = p->kap_num, Q = p->kap_den;
        i128 a0 = Q > P ? (Q - 1 - P) / (2 * P) : 0;
        if (a0 > cap) a0 = cap;
        A = (int64_t)a0;
        if (!room(A)) {                                    // headroom binds first: bisect it
            int64_t lo_ok = 0, hi_bad = A;
            while (hi_bad - lo_ok > 1) {
                const int64_t mid = lo_ok + (hi_bad - lo_ok) / 2;
                (room(mid) ? lo_ok : hi_bad) = mid;
            }
            return lo_ok;
        }
    }
    int64_t ppp = host_phi(p->hp, A, rd), pmp = host_phi(p->hm, A, rd);
    int64_t ppn = host_phi(p->hp, -A, rd), pmn = host_phi(p->hm, -A, rd);
    const int64_t stop = A + ((int64_t)1 << 24) < cap ? A + ((int64_t)1 << 24) : cap;
    while (A < stop) {
        const int64_t a1 = A + 1;
        const int64_t pp1 = host_phi(p->hp, a1, rd), pm1 = host_phi(p->hm, a1, rd);
        const int64_t ppm = host_phi(p->hp, -a1, rd), pmm = host_phi(p->hm, -a1, rd);
        const int64_t dp = pp1 - ppp, dm = pm1 - pmp;            // step A -> A+1
        const int64_t dpn = ppn - ppm, dmn = pmn - pmm;          // step -A-1 -> -A
        if (dp < 0 || dm > 0 || dp - dm > 1 || dpn < 0 || dmn > 0 || dpn - dmn > 1) break;
        if (!room(a1)) break;
        ppp = pp1; pmp = pm1; ppn = ppm; pmn = pmm;
        A = a1;
    }
    return A;
}

static int build_rule(fqnm_plan_t* p)
{
    fqnm_plan_desc& d = p->d;
    // two-point kinds (Thm P:262-280) reuse the rule builder of their split
    // counterpart for kappa, coefficients and the admissible range
    const int tp_kind = (d.flux_kind == FQNM_BURGERS_GODUNOV || d.flux_kind == FQNM_BURGERS_EO2 ||
                         d.flux_kind == FQNM_BURGERS_LF2) ? d.flux_kind : 0;
    const int kind = tp_kind == FQNM_BURGERS_LF2 ? FQNM_BURGERS_LF
                   : tp_kind ? FQNM_BURGERS_EO : d.flux_kind;
    int64_t P = d.kappa_num, Q = d.kappa_den;
    if (kind == FQNM_LINEAR || kind == FQNM_BURGERS_EO) {
        if (P == 0 && Q == 0) {
            double a = d.flux_param == 0.0 ? 1.0 : d.flux_param;
            double kd = (kind == FQNM_LINEAR) ? a * d.dt_dx : d.delta * d.dt_dx / 2.0;
            if (!rationalize(kd, &P, &Q))
                return fail(FQNM_ERR_ARG, "kappa = %.17g has no exact rational with "
                            "denominator <= 2^31 (pass kappa_num/kappa_den)", kd);
        } else {
            if (Q <= 0 || P == 0) return fail(FQNM_ERR_ARG, "kappa_den must be > 0, kappa_num != 0");
            int64_t g = gcd64(P, Q);
            P /= g; Q /= g;
        }
        p->kap_num = P;
        p->kap_den = Q;
        if (kind == FQNM_LINEAR) {
            HostMap m;
            m.c2 = 0; m.c1 = P; m.den = Q; m.supp = SUPP_ALL;
            if (P > 0) { p->hp = m; p->hm = HostMap(); }
            else { p->hm = m; p->hp = HostMap(); }
        } else {
            if (P < 0) return fail(FQNM_ERR_ARG, "Burgers EO needs delta*dt_dx > 0");
            HostMap a, b;
            a.c2 = P; a.c1 = 0; a.den = Q; a.supp = SUPP_POS;
            b.c2 = P; b.c1 = 0; b.den = Q; b.supp = SUPP_NEG;
            p->hp = a; p->hm = b;
        }
    } else if (kind == FQNM_BURGERS_LF) {
        // f+- = (u^2/2 +- alpha u)/2  ->  phi+- = round(k2 q^2 +- k1 q), k2 = delta lam/4, k1 = alpha lam/2
        if (!(d.flux_param > 0)) return fail(FQNM_ERR_ARG, "Burgers LF needs flux_param alpha > 0");
        int64_t P2, Q2, P1, Q1;
        if (!rationalize(d.delta * d.dt_dx / 4.0, &P2, &Q2) ||
            !rationalize(d.flux_param * d.dt_dx / 2.0, &P1, &Q1))
            return fail(FQNM_ERR_ARG, "LF coefficients have no exact rational form");
        int64_t g = gcd64(Q1, Q2);
        i128 den = (i128)Q1 / g * Q2;
        i128 c2 = (i128)P2 * (den / Q2), c1 = (i128)P1 * (den / Q1);
        if (den > INT64_MAX / 4 || c2 > INT64_MAX / 4 || c1 > INT64_MAX / 4)
            return fail(FQNM_ERR_UNSUPPORTED, "LF coefficients too large for int64");
        HostMap a, b;
        a.c2 = (int64_t)c2; a.c1 = (int64_t)c1; a.den = (int64_t)den; a.supp = SUPP_ALL;
        b.c2 = (int64_t)c2; b.c1 = -(int64_t)c1; b.den = (int64_t)den; b.supp = SUPP_ALL;
        p->hp = a; p->hm = b;
        p->kap_num = P2; p->kap_den = Q2;
    } else {
        return fail(FQNM_ERR_ARG, "unknown flux kind %d", kind);
    }
    p->dep_left = !map_is_zero(p->hp);
    p->dep_right = !map_is_zero(p->hm);

    // ---- range, D8, fast-path selection ----
    const bool lin_half = (kind == FQNM_LINEAR && P == 1 && Q == 2 &&
                           d.rounding == FQNM_ROUND_HALF_AWAY);
    bool eo_fast_ok = false;
    int64_t a_fast = 0;
    if (kind == FQNM_BURGERS_EO && d.rounding == FQNM_ROUND_HALF_AWAY && P >= 1 &&
        P < (1 << 29) && Q < (1 << 29)) {
        // maps.cuh eo_g: exact for |q| < 2^22 and P q^2 / Q <= 2^20
        double am = std::sqrt(std::ldexp(1.0, 20) * (double)Q / (double)P);
        a_fast = (int64_t)am + 1;
        while (a_fast > 0 && (i128)P * a_fast * a_fast > ((i128)1 << 20) * Q) --a_fast;
        if (a_fast > (1 << 22) - 1) a_fast = (1 << 22) - 1;
        eo_fast_ok = a_fast > 0;
    }
    int64_t lo = d.q_lo, hi = d.q_hi;
    const int64_t i32lo = INT32_MIN + 1, i32hi = INT32_MAX;
    if (kind == FQNM_LINEAR) {
        // D8 holds on all of Z iff |kappa| <= 1 (increments of round(kappa q) are 0/1)
        const int64_t aP = P < 0 ? -P : P;
        if (aP > Q)
            return fail(FQNM_ERR_CFL, "linear |kappa| = %lld/%lld > 1 violates D8", (long long)P,
                        (long long)Q);
        // R_LIN_FAST domain (maps.cuh lin_phi): |q| < 2^24, |kappa q| <= 2^20, Q < 2^29
        int64_t a_lin = 0;
        if (!lin_half && d.rounding == FQNM_ROUND_HALF_AWAY && Q < (1 << 29)) {
            a_lin = (int64_t)(((i128)1 << 20) * Q / aP);
            if (a_lin > (1 << 24) - 1) a_lin = (1 << 24) - 1;
        }
        const bool derive = (lo == 0 && hi == 0);
        if (derive) {
            if (a_lin > 0 && d.check_range) { lo = -a_lin; hi = a_lin; }   // checked at every step
            else { lo = i32lo; hi = i32hi; }
        }
        if (lo < i32lo || hi > i32hi) return fail(FQNM_ERR_RANGE, "range exceeds int32 state");
        const int64_t amax = (lo < 0 ? -lo : lo) > hi ? (lo < 0 ? -lo : lo) : hi;
        if (lin_half) p->rule = R_LIN_HALF;
        else if (a_lin > 0 && amax <= a_lin) p->rule = R_LIN_FAST;
        else {
            if (!(generic_headroom(p->hp, amax) && generic_headroom(p->hm, amax)))
                return fail(FQNM_ERR_RANGE, "int64 headroom exceeded");
            p->rule = R_GENERIC;
        }
    } else {
        if (lo == 0 && hi == 0) {
            // derive the largest symmetric range on which D8 holds
            int64_t A = d8_symmetric_limit(p, kind == FQNM_BURGERS_EO);
            if (eo_fast_ok && A > a_fast) {
                // the fast closed form is exact only on |q| <= a_fast: that is the plan's
                // range; range-checked steps beyond it fall back to the int64 rule
                if (A >= 1) p->d8_lim = A;
                A = a_fast;
            }
            if (A < 1) return fail(FQNM_ERR_CFL, "D8 fails already at |q| <= 1");
            lo = -A; hi = A;
        } else {
            if (lo >= hi) return fail(FQNM_ERR_ARG, "q_lo must be < q_hi");
            if (lo < i32lo || hi > i32hi) return fail(FQNM_ERR_RANGE, "range exceeds int32 state");
            if (!p->trusted_range) {
                if (hi - lo > ((int64_t)1 << 27))
                    return fail(FQNM_ERR_UNSUPPORTED, "declared range too wide to validate D8");
                int64_t bad = d8_first_violation(p, lo, hi);
                if (bad >= lo)
                    return fail(FQNM_ERR_CFL, "D8 (integer monotonicity) fails at q = %lld", (long long)bad);
            }
            int64_t amax = (lo < 0 ? -lo : lo) > hi ? (lo < 0 ? -lo : lo) : hi;
            if (!generic_headroom(p->hp, amax) || !generic_headroom(p->hm, amax))
                return fail(FQNM_ERR_RANGE, "int64 headroom exceeded on the declared range");
        }
        int64_t amax = (lo < 0 ? -lo : lo) > hi ? (lo < 0 ? -lo : lo) : hi;
        p->rule = (eo_fast_ok && amax <= a_fast) ? (P == 1 ? R_EO_P1 : R_EO_FAST) : R_GENERIC;
    }
    int tp_fast = 0;
    if (tp_kind) {
        // Phi = round(num/den), num = the two maps' numerators combined (max for Godunov):
        // |num| <= 2 (|c2| a^2 + |c1| a) on the range; int64 headroom for round_div_i64
        const int64_t amax = (lo < 0 ? -lo : lo) > hi ? (lo < 0 ? -lo : lo) : hi;
        const HostMap& m = p->hp;
        i128 A = amax;
        i128 num = 2 * ((i128)(m.c2 < 0 ? -m.c2 : m.c2) * A * A + (i128)(m.c1 < 0 ? -m.c1 : m.c1) * A);
        if (2 * num + m.den >= ((i128)1 << 62))
            return fail(FQNM_ERR_RANGE, "int64 headroom exceeded for the two-point rule");
        // Godunov on the EO fast path's domain: Phi = g(max(max(qL,0), -min(qR,0))) with the
        // EO magnitude g(x) = RHA(kappa x^2) evaluated by the closed form (maps.cuh)
        tp_fast = (tp_kind == FQNM_BURGERS_GODUNOV && (p->rule == R_EO_P1 || p->rule == R_EO_FAST))
                      ? (p->rule == R_EO_P1 ? 1 : 2) : 0;
        p->rule = tp_fast ? R_TP_FAST : R_TWOPOINT;
        p->dep_left = p->dep_right = true;
    }
    p->lo = lo;
    p->hi = hi;

    DevRule& r = p->dr;
    std::memset(&r, 0, sizeof r);
    r.c2p = p->hp.c2; r.c1p = p->hp.c1; r.denp = p->hp.den; r.suppp = p->hp.supp;
    r.c2m = p->hm.c2; r.c1m = p->hm.c1; r.denm = p->hm.den; r.suppm = p->hm.supp;
    if (map_is_zero(p->hp)) r.suppp = SUPP_NONE;
    if (map_is_zero(p->hm)) r.suppm = SUPP_NONE;
    r.rounding = d.rounding;
    r.one = 1;
    r.mone = -1;
    r.lin_minus = (kind == FQNM_LINEAR && P < 0) ? 1 : 0;
    if (p->rule == R_LIN_FAST) {
        const int64_t aP = P < 0 ? -P : P;
        r.eo_ntwoP = (int32_t)(-2 * aP);
        r.eo_twoQ = (int32_t)(2 * Q);
        r.eo_c1 = (int32_t)(uint32_t)((uint64_t)(Q - 1) - (uint64_t)(2 * Q) * 0x4B400000ull);
        const double target = ((double)aP / (double)Q) * (1.0 - std::ldexp(1.0, -21));
        float cf = (float)target;
        while ((double)cf > target) cf = std::nextafterf(cf, 0.0f);
        r.eo_cf = cf;
    }
    if (p->rule == R_TWOPOINT || p->rule == R_TP_FAST) {
        r.tp_kind = tp_kind;
        r.tp_c2 = p->hp.c2;
        r.tp_c1 = tp_kind == FQNM_BURGERS_LF2 ? p->hp.c1 : 0;
        r.tp_den = p->hp.den;
        r.tp_fast = tp_fast;
    }
    // round(num / den) in float64 (maps.cuh round_div_dp): RHA, den > 0 and |num| < 2^44 on the
    // admissible range; otherwise the int64 division stays
    {
        auto dv_set = [&](int which, int64_t den, i128 num_bound) {
            r.dv_ok[which] = 0;
            if (d.rounding != FQNM_ROUND_HALF_AWAY || den <= 0 || num_bound >= ((i128)1 << 44)) return;
            const long double inv = (1.0L / (long double)den) * (1.0L + std::ldexp(1.0L, -46));
            double dv = (double)inv;
            uint64_t bits;
            std::memcpy(&bits, &dv, sizeof bits);
            bits &= ~3ull;                               // 1.5 * dv must be exact: 3 (m / 4) < 2^53
            std::memcpy(&dv, &bits, sizeof bits);
            r.dv_inv[which] = dv;
            r.dv_c[which] = -(std::ldexp(dv, 52) + std::ldexp(dv, 51));
            r.dv_ok[which] = 1;
        };
        const bool bounded = p->lo > INT64_MIN / 2 && p->hi < INT64_MAX / 2;
        const i128 A = bounded ? (i128)std::max(std::llabs((long long)p->lo), std::llabs((long long)p->hi))
                               : ((i128)1 << 40);
        auto map_bound = [&](const HostMap& m) {
            return (i128)(m.c2 < 0 ? -m.c2 : m.c2) * A * A + (i128)(m.c1 < 0 ? -m.c1 : m.c1) * A;
        };
        dv_set(0, p->hp.den, map_bound(p->hp));
        dv_set(1, p->hm.den, map_bound(p->hm));
        if (tp_kind) dv_set(2, p->hp.den, 2 * map_bound(p->hp));
    }
    if (p->rule == R_EO_FAST || p->rule == R_EO_P1 || tp_fast) {
        r.eo_ntwoP = (int32_t)(-2 * P);
        r.eo_twoQ = (int32_t)(2 * Q);
        r.eo_c1 = (int32_t)(uint32_t)((uint64_t)(Q - 1) - (uint64_t)(2 * Q) * 0x4B400000ull);
        r.eo_nQ = (int32_t)(-Q);
        r.eo_c6 = (int32_t)(uint32_t)((uint64_t)Q * 0x4B400001ull - (uint64_t)((Q + 1) / 2));
        r.eo_P = (int32_t)P;
        // largest float <= kappa (1 - 2^-21): a strict relative underestimate of kappa
        const double target = ((double)P / (double)Q) * (1.0 - std::ldexp(1.0, -21));
        float cf = (float)target;
        while ((double)cf > target) cf = std::nextafterf(cf, 0.0f);
        r.eo_cf = cf;
        // float64 form (eo_g_dp): see maps.cuh for the exactness argument
        const long double inv = ((long double)P / (long double)Q) * (1.0L + std::ldexp(1.0L, -46));
        r.eo_dinv = (double)inv;
        r.eo_dc1 = -std::ldexp(r.eo_dinv, 52);
        r.eo_xoff = (long long)(1023 + 52) << 52;       // bits of 2^52: one ulp is 1
        const long double qm = (long double)std::max(std::llabs((long long)p->lo), std::llabs((long long)p->hi));
        r.eo_dp_ok = ((long double)P * qm * qm < std::ldexp(1.0L, 44)) ? 1 : 0;
        // the P = 1 stepping kernels use the float64 form unconditionally; its condition holds
        // on the whole fast-path domain (|q| < 2^22), but fall back to the general-P rule
        // (float32 + integer remainder) should a range ever exceed it
        if (p->rule == R_EO_P1 && !r.eo_dp_ok) p->rule = R_EO_FAST;
    }
    return FQNM_OK;
}

// ---------------------------------------------------------------------------
static int resident_geometry(const fqnm_plan_t* p, int k, int* P, int* base, int* rem, int* H);

static int choose_kernel(fqnm_plan_t* p)
{
    const fqnm_plan_desc& d = p->d;
    if (d.nvar == 3) {
        p->family = 5;
        // V = 2 (64-cell windows, 151 registers, 12 warps/SM) since the branch-free interior
        // path: cfg5 80.8 vs 70.4 (V = 1) vs 71.7 (V = 4) GCUPS; small problems keep V = 1
        // (twice the warps)
        p->V = (d.n_local * (d.batch > 0 ? d.batch : 1) >= (1 << 17)) ? 2 : 1;
        p->k = 1;
        return FQNM_OK;
    }
    const int64_t n = d.n_local;
    if (d.boundary == FQNM_HALO) {
        p->family = 2;
    } else if (n % 32 == 0 && warp_ensemble_has_V((int)(n / 32)) && n <= 1024) {
        p->family = 3;
        p->V = (int)(n / 32);
    } else if (n <= 16384) {
        p->family = 4;
    } else if (d.batch == 1 && n <= RESIDENT_MAX_CELLS) {
        p->family = 6;                  // one mid-size problem: whole domain resident on chip
        p->V = 8;
        p->k = d.k;
        if (p->k <= 0) {
            // time per step ~ (warps per SM sub-partition) x t_step + t_exchange / k: the
            // exchange (one L2 round trip, ~2.7 us) is paid once per k steps, but a deeper
            // halo means more warps (P = n / (256 - 2k)), and past 4 x 148 warps some
            // sub-partitions issue for two.  cfg2: k = 72 gives P = 586 (one warp per
            // sub-partition, 128-thread CTAs), k = 80 gave P = 683 in 86 CTAs of 8 warps
            // (2.65 -> 1.9 ms; profiles/r02_tune_cfg2.jsonl)
            double best = 1e30;
            int bestk = 0;
            for (int kk = 124; kk >= 8; kk -= 4) {
                int P, base, rem, H;
                if (resident_geometry(p, kk, &P, &base, &rem, &H) != FQNM_OK) continue;
                const int wps = (P + 148 * 4 - 1) / (148 * 4);
                const double t = wps * 50.0 + 2700.0 / kk;
                if (t < best) { best = t; bestk = kk; }
            }
            p->k = bestk > 0 ? bestk : 16;
        }
    } else {
        p->family = 2;
    }
    if (p->family == 2) {
        const bool two = p->dep_left && p->dep_right;
        if (p->rule == R_LIN_HALF) { p->V = 32; p->k = 64; p->minb = 2; }
        else if (p->rule == R_EO_FAST || p->rule == R_EO_P1 || p->rule == R_TP_FAST) {
            p->V = 32; p->k = p->rule == R_TP_FAST ? 24 : 32; p->minb = 2;   // EO: sweep r02_tune_sign.jsonl
        }
        else { p->V = 8; p->k = two ? 8 : 16; }
        if (d.k > 0) p->k = d.k;
        if (d.boundary == FQNM_HALO && p->k > d.halo) p->k = (int)d.halo;
    }
    return FQNM_OK;
}

static int round4(int x) { return (x + 3) & ~3; }


static int resident_geometry(const fqnm_plan_t* p, int k, int* P, int* base, int* rem, int* H)
{
    const int W = 32 * p->V;
    *H = round4(k);
    const int S = W - 2 * *H;
    if (S < *H || S < 4) return FQNM_ERR_ARG;
    const int64_t n = p->d.n_local;
    int64_t P64 = (n + S - 1) / S;
    if (P64 > RESIDENT_MAX_WARPS) return FQNM_ERR_UNSUPPORTED;
    *P = (int)P64;
    *base = (int)(n / P64);
    *rem = (int)(n % P64);
    if (*base < *H) return FQNM_ERR_ARG;
    return FQNM_OK;
}

static int resident_alloc(fqnm_plan_t* p)
{
    int P, base, rem, H;
    int rc = resident_geometry(p, p->k, &P, &base, &rem, &H);
    if (rc != FQNM_OK)
        return fail(rc, "resident stepper geometry invalid for n = %lld", (long long)p->d.n_local);
    const int Hmax = 124;                    // largest halo any allowed k needs
    // edges sized for the smallest S (largest P) any allowed k produces
    const int64_t n = p->d.n_local;
    int64_t Pmax = (n + 4 - 1) / 4;
    if (Pmax > RESIDENT_MAX_WARPS) Pmax = RESIDENT_MAX_WARPS;
    if (!p->edges) {                         // 8-byte {value, tag} words (K6 exchange)
        const size_t eb = sizeof(uint64_t) * 2 * Pmax * 2 * (size_t)Hmax;
        CUDA_TRY(cudaMalloc(&p->edges, eb));
        CUDA_TRY(cudaMemset(p->edges, 0, eb));                              // tag 0 never matches
    }
    if (!p->flags) {
        CUDA_TRY(cudaMalloc(&p->flags, sizeof(unsigned int) * Pmax));
        CUDA_TRY(cudaMemset(p->flags, 0, sizeof(unsigned int) * Pmax));   // tags start at 1
        p->tag_base = 1;
    }
    p->res_P = (int)Pmax;
    return FQNM_OK;
}

// largest steps per block the geometry of V admits
static int max_block_steps(const fqnm_plan_t* p, int V)
{
    const int W = 32 * V;
    const int sides = (p->dep_left ? 1 : 0) + (p->dep_right ? 1 : 0);
    if (sides == 0) return 1 << 30;
    // keep at least W/4 useful cells per window
    int k = (W - W / 4) / sides;
    return k & ~3;
}

static int plan_build(fqnm_plan_t** out, const fqnm_plan_desc* din, bool allocate, bool trusted_range)
{
    if (!out || !din) return fail(FQNM_ERR_ARG, "null argument");
    *out = nullptr;
    const fqnm_plan_desc& d = *din;
    if (d.n_local < 2) return fail(FQNM_ERR_ARG, "n_local must be >= 2");
    if (d.batch < 1) return fail(FQNM_ERR_ARG, "batch must be >= 1");
    if (!(std::isfinite(d.delta) && d.delta > 0)) return fail(FQNM_ERR_ARG, "delta must be finite and > 0");
    if (!(std::isfinite(d.dt_dx) && d.dt_dx > 0)) return fail(FQNM_ERR_ARG, "dt_dx must be finite and > 0");
    if (d.boundary < 0 || d.boundary > 2) return fail(FQNM_ERR_ARG, "unknown boundary %d", d.boundary);
    if (d.rounding < 0 || d.rounding > 2) return fail(FQNM_ERR_ARG, "unknown rounding %d", d.rounding);
    fqnm_plan_t* p = new (std::nothrow) fqnm_plan_t();
    if (!p) return fail(FQNM_ERR_NOMEM, "out of host memory");
    p->trusted_range = trusted_range;
    p->d = d;
    p->d.n_global = d.n_global ? d.n_global : d.n_local;
    p->st = (cudaStream_t)d.stream;
    int rc;
    if (d.flux_kind == FQNM_EULER_ROE || d.flux_kind == FQNM_EULER_ROE_DENSITY) {
        if (d.nvar != 3 || d.dtype != FQNM_I64) {
            delete p;
            return fail(FQNM_ERR_ARG, "Euler plans need nvar = 3 and dtype = FQNM_I64");
        }
        if (d.boundary == FQNM_HALO) { delete p; return fail(FQNM_ERR_UNSUPPORTED, "Euler split domains"); }
        double gamma = d.flux_param == 0.0 ? 1.4 : d.flux_param;
        if (!(gamma > 1.0)) { delete p; return fail(FQNM_ERR_ARG, "gamma must be > 1"); }
        p->s_e = d.dt_dx / d.delta;          // s = fl(dt/dx / delta)
        p->g1_e = gamma - 1.0;                // g1 = fl(gamma - 1)
        p->lo = INT64_MIN;
        p->hi = INT64_MAX;
    } else {
        if (d.nvar != 1 || d.dtype != FQNM_I32) {
            delete p;
            return fail(FQNM_ERR_UNSUPPORTED, "scalar plans need nvar = 1 and dtype = FQNM_I32");
        }
        if ((rc = build_rule(p)) != FQNM_OK) { delete p; return rc; }
    }
    if (d.boundary == FQNM_HALO) {
        if (d.halo < 4 || d.halo % 4 != 0) { delete p; return fail(FQNM_ERR_ARG, "halo must be a positive multiple of 4"); }
        if (d.batch != 1) { delete p; return fail(FQNM_ERR_UNSUPPORTED, "split domains with batch > 1"); }
    }
    choose_kernel(p);
    if (p->family == 2) {
        int kmax = max_block_steps(p, p->V);
        if (p->k > kmax) p->k = kmax;
        if (p->k < 1) p->k = 1;
    }
    if (!allocate) {
        *out = p;
        return FQNM_OK;
    }
    // device buffers
    cudaError_t e;
    if (d.boundary == FQNM_HALO && d.p2p) {
        const size_t bytes = state_elems(p->d) * elem_size(p->d);
        for (int i = 0; i < 2; ++i) {
            if ((e = cudaMalloc(&p->hbuf[i], bytes)) != cudaSuccess) {
                fqnm_destroy(p);
                return fail(FQNM_ERR_NOMEM, "cudaMalloc halo buffer: %s", cudaGetErrorString(e));
            }
            cudaMemset(p->hbuf[i], 0, bytes);
        }
        if ((e = cudaMalloc(&p->hflags, 2 * sizeof(unsigned int))) != cudaSuccess) {
            fqnm_destroy(p);
            return fail(FQNM_ERR_NOMEM, "cudaMalloc halo flags: %s", cudaGetErrorString(e));
        }
        cudaMemset(p->hflags, 0, 2 * sizeof(unsigned int));
    }
    if (p->family == 6) {
        int rc6 = resident_alloc(p);
        if (rc6 != FQNM_OK) { fqnm_destroy(p); return rc6; }
    }
    if (p->family == 2 || p->family == 1 || p->family == 5 || p->family == 6) {
        if (d.boundary != FQNM_HALO) {
            p->scratch_bytes = state_elems(p->d) * elem_size(p->d);
            e = cudaMalloc(&p->scratch, p->scratch_bytes);
            if (e != cudaSuccess) {
                delete p;
                return fail(FQNM_ERR_NOMEM, "cudaMalloc(%zu) scratch: %s", (size_t)state_elems(d) * elem_size(d),
                            cudaGetErrorString(e));
            }
        }
    }
    if ((e = cudaMalloc(&p->d_minmax, 2 * sizeof(long long))) != cudaSuccess ||
        (e = cudaMallocHost(&p->h_minmax, 4 * sizeof(long long))) != cudaSuccess) {
        fqnm_destroy(p);
        return fail(FQNM_ERR_CUDA, "allocating range-check buffers: %s", cudaGetErrorString(e));
    }
    *out = p;
    return FQNM_OK;
}

extern "C" int fqnm_plan_ex(fqnm_plan_t** out, const fqnm_plan_desc* din)
{
    return plan_build(out, din, true);
}

extern "C" int fqnm_plan(fqnm_plan_t** out, int64_t N, double delta, double dt_dx, int flux_kind,
                         int boundary)
{
    fqnm_plan_desc d;
    fqnm_desc_init(&d);
    d.n_local = N;
    d.n_global = N;
    d.delta = delta;
    d.dt_dx = dt_dx;
    d.flux_kind = flux_kind;
    d.boundary = boundary;
    d.check_range = 1;
    if (boundary != FQNM_PERIODIC && boundary != FQNM_TRANSMISSIVE)
        return fail(FQNM_ERR_ARG, "fqnm_plan: boundary must be PERIODIC or TRANSMISSIVE");
    if (flux_kind == FQNM_EULER_ROE || flux_kind == FQNM_EULER_ROE_DENSITY) {
        d.nvar = 3;
        d.dtype = FQNM_I64;
        d.flux_param = 1.4;
        d.check_range = 0;
    }
    return fqnm_plan_ex(out, &d);
}

// multi-D admissible range: see the 2D/3D range guard below
static void md_clamp_range(fqnm_plan_t* p, int dims)
{
    const int64_t lim = (int64_t)INT32_MAX / (1 + 4 * dims);
    if (p->hi > lim) p->hi = lim;
    if (p->lo < -lim) p->lo = -lim;
}

extern "C" int fqnm_plan_2d(fqnm_plan_t** out, int64_t nx, int64_t ny, double delta, double dt_dx,
                            double dt_dy, int flux_kind, int boundary, double param_x, double param_y)
{
    if (!out) return fail(FQNM_ERR_ARG, "null argument");
    *out = nullptr;
    if (nx < 2 || ny < 2) return fail(FQNM_ERR_ARG, "nx and ny must be >= 2");
    if (flux_kind != FQNM_LINEAR && flux_kind != FQNM_BURGERS_EO && flux_kind != FQNM_BURGERS_LF)
        return fail(FQNM_ERR_UNSUPPORTED, "2D plans support the scalar flux kinds");
    if (boundary != FQNM_PERIODIC && boundary != FQNM_TRANSMISSIVE)
        return fail(FQNM_ERR_ARG, "2D plans: boundary must be PERIODIC or TRANSMISSIVE");
    if (!(std::isfinite(dt_dy) && dt_dy > 0)) return fail(FQNM_ERR_ARG, "dt_dy must be finite and > 0");
    fqnm_plan_desc d;
    fqnm_desc_init(&d);
    d.n_local = nx * ny;
    d.n_global = nx * ny;
    d.delta = delta;
    d.dt_dx = dt_dy;
    d.flux_kind = flux_kind;
    d.boundary = boundary;
    d.flux_param = param_y;
    d.check_range = 1;
    // y rule (host-only build)
    fqnm_plan_t* py = nullptr;
    int rc = plan_build(&py, &d, false);
    if (rc != FQNM_OK) return rc;
    // x rule + the plan
    d.dt_dx = dt_dx;
    d.flux_param = param_x;
    fqnm_plan_t* p = nullptr;
    rc = plan_build(&p, &d, false);
    if (rc != FQNM_OK) { delete py; return rc; }
    p->nx = nx;
    p->ny = ny;
    p->hpy = py->hp;
    p->hmy = py->hm;
    p->dry = py->dr;
    p->same_xy = std::memcmp(&p->dr, &py->dr, sizeof(DevRule)) == 0;
    if (p->rule != py->rule) p->rule = R_GENERIC;          // both directions on the int64 path
    p->lo = p->lo > py->lo ? p->lo : py->lo;
    p->hi = p->hi < py->hi ? p->hi : py->hi;
    md_clamp_range(p, 2);
    p->dep_left = p->dep_left || py->dep_left;
    p->dep_right = p->dep_right || py->dep_right;
    delete py;
    p->family = 7;
    p->V = 0;
    p->k = STEP2D_KMAX;
    p->scratch_bytes = state_elems(p->d) * elem_size(p->d);
    cudaError_t e;
    if ((e = cudaMalloc(&p->scratch, p->scratch_bytes)) != cudaSuccess ||
        (e = cudaMalloc(&p->d_minmax, 2 * sizeof(long long))) != cudaSuccess ||
        (e = cudaMallocHost(&p->h_minmax, 4 * sizeof(long long))) != cudaSuccess ||
        (e = cudaMalloc(&p->md_guard, sizeof(int))) != cudaSuccess ||
        (e = cudaMallocHost(&p->md_guard_host, sizeof(int))) != cudaSuccess) {
        fqnm_destroy(p);
        return fail(FQNM_ERR_NOMEM, "allocating 2D plan buffers: %s", cudaGetErrorString(e));
    }
    *out = p;
    return FQNM_OK;
}

extern "C" int fqnm_plan_3d(fqnm_plan_t** out, int64_t nx, int64_t ny, int64_t nz, double delta,
                            double dt_dx, double dt_dy, double dt_dz, int flux_kind, int boundary,
                            double param_x, double param_y, double param_z)
{
    if (!out) return fail(FQNM_ERR_ARG, "null argument");
    *out = nullptr;
    if (nx < 2 || ny < 2 || nz < 2) return fail(FQNM_ERR_ARG, "nx, ny and nz must be >= 2");
    if (nx > ((int64_t)1 << 31) / ny / nz) return fail(FQNM_ERR_ARG, "nx * ny * nz must be < 2^31");
    if (flux_kind != FQNM_LINEAR && flux_kind != FQNM_BURGERS_EO && flux_kind != FQNM_BURGERS_LF)
        return fail(FQNM_ERR_UNSUPPORTED, "3D plans support the split scalar flux kinds");
    if (boundary != FQNM_PERIODIC && boundary != FQNM_TRANSMISSIVE)
        return fail(FQNM_ERR_ARG, "3D plans: boundary must be PERIODIC or TRANSMISSIVE");
    if (!(std::isfinite(dt_dy) && dt_dy > 0 && std::isfinite(dt_dz) && dt_dz > 0))
        return fail(FQNM_ERR_ARG, "dt_dy and dt_dz must be finite and > 0");
    fqnm_plan_desc d;
    fqnm_desc_init(&d);
    d.n_local = nx * ny * nz;
    d.n_global = d.n_local;
    d.delta = delta;
    d.flux_kind = flux_kind;
    d.boundary = boundary;
    d.check_range = 1;
    // per-direction rules (host-only builds), then the plan with the x rule
    fqnm_plan_t* pd[3] = {nullptr, nullptr, nullptr};
    const double lam[3] = {dt_dx, dt_dy, dt_dz}, par[3] = {param_x, param_y, param_z};
    for (int m = 2; m >= 0; --m) {
        d.dt_dx = lam[m];
        d.flux_param = par[m];
        int rc = plan_build(&pd[m], &d, false);
        if (rc != FQNM_OK) {
            for (int j = 0; j < 3; ++j) delete pd[j];
            return rc;
        }
    }
    fqnm_plan_t* p = pd[0];
    p->nx = nx;
    p->ny = ny;
    p->nz = nz;
    p->dry = pd[1]->dr;
    p->drz = pd[2]->dr;
    p->same_xy = std::memcmp(&p->dr, &pd[1]->dr, sizeof(DevRule)) == 0 &&
                 std::memcmp(&p->dr, &pd[2]->dr, sizeof(DevRule)) == 0;
    for (int m = 1; m < 3; ++m) {
        if (p->rule != pd[m]->rule) p->rule = R_GENERIC;     // all directions on the int64 path
        p->lo = p->lo > pd[m]->lo ? p->lo : pd[m]->lo;
        p->hi = p->hi < pd[m]->hi ? p->hi : pd[m]->hi;
        delete pd[m];
    }
    md_clamp_range(p, 3);
    p->family = 8;
    p->V = 0;
    p->k = 1;
    p->scratch_bytes = state_elems(p->d) * elem_size(p->d);
    cudaError_t e;
    if ((e = cudaMalloc(&p->scratch, p->scratch_bytes)) != cudaSuccess ||
        (e = cudaMalloc(&p->d_minmax, 2 * sizeof(long long))) != cudaSuccess ||
        (e = cudaMallocHost(&p->h_minmax, 4 * sizeof(long long))) != cudaSuccess ||
        (e = cudaMalloc(&p->md_guard, sizeof(int))) != cudaSuccess ||
        (e = cudaMallocHost(&p->md_guard_host, sizeof(int))) != cudaSuccess) {
        fqnm_destroy(p);
        return fail(FQNM_ERR_NOMEM, "allocating 3D plan buffers: %s", cudaGetErrorString(e));
    }
    *out = p;
    return FQNM_OK;
}

static void pipe_release(fqnm_plan_t* p)
{
    for (int i = 1; i < 4; ++i) {
        if (p->pipe_kids[i]) fqnm_destroy(p->pipe_kids[i]);
        p->pipe_kids[i] = nullptr;
    }
    if (p->pipe_child) fqnm_destroy(p->pipe_child);
    p->pipe_child = nullptr;
    p->pipe_kids[0] = nullptr;
    p->pipe_start.clear();
    p->pipe_size.clear();
    for (int i = 0; i < 3; ++i) {
        if (p->pipe_buf[i]) cudaFree(p->pipe_buf[i]);
        p->pipe_buf[i] = nullptr;
    }
    if (p->pipe_head) cudaFree(p->pipe_head);
    p->pipe_head = nullptr;
    if (p->pipe_sign) cudaFree(p->pipe_sign);
    p->pipe_sign = nullptr;
    if (p->pipe_sign_host) cudaFreeHost(p->pipe_sign_host);
    p->pipe_sign_host = nullptr;
    if (p->pipe_guard) cudaFree(p->pipe_guard);
    if (p->pipe_guard_host) cudaFreeHost(p->pipe_guard_host);
    p->pipe_guard = nullptr;
    p->pipe_guard_host = nullptr;
    for (cudaEvent_t& e : p->pipe_ev)
        if (e) { cudaEventDestroy(e); e = nullptr; }
    if (p->pipe_h2d) cudaStreamDestroy(p->pipe_h2d);
    if (p->pipe_d2h) cudaStreamDestroy(p->pipe_d2h);
    p->pipe_h2d = p->pipe_d2h = nullptr;
    p->pipe_H = p->pipe_C = p->pipe_m = 0;
}

extern "C" void fqnm_destroy(fqnm_plan_t* p)
{
    if (!p) return;
    cudaStreamSynchronize(p->st);
    if (p->generic_child) fqnm_destroy(p->generic_child);
    if (p->scratch) cudaFree(p->scratch);
    if (p->d_minmax) cudaFree(p->d_minmax);
    if (p->h_minmax) cudaFreeHost(p->h_minmax);
    if (p->e2e_dev) cudaFree(p->e2e_dev);
    if (p->ens_h2d) cudaStreamDestroy(p->ens_h2d);
    if (p->ens_d2h) cudaStreamDestroy(p->ens_d2h);
    for (cudaEvent_t e : p->ens_ev)
        if (e) cudaEventDestroy(e);
    if (p->edges) cudaFree(p->edges);
    if (p->flags) cudaFree(p->flags);
    for (int i = 0; i < 2; ++i)
        if (p->hbuf[i]) cudaFree(p->hbuf[i]);
    if (p->hflags) cudaFree(p->hflags);
    if (p->pflags) cudaFree(p->pflags);
    if (p->pcounter) cudaFree(p->pcounter);
    if (p->md_guard) cudaFree(p->md_guard);
    if (p->md_guard_host) cudaFreeHost(p->md_guard_host);
    for (cudaEvent_t e : p->ev) cudaEventDestroy(e);
    pipe_release(p);
    delete p;
}

extern "C" int fqnm_set_stream(fqnm_plan_t* p, void* stream)
{
    if (!p) return fail(FQNM_ERR_ARG, "null plan");
    p->st = (cudaStream_t)stream;
    return FQNM_OK;
}

static bool aligned16(const void* x) { return ((uintptr_t)x & 15u) == 0; }

// ---------------------------------------------------------------------------
static int check_range(fqnm_plan_t* p, const void* q, bool* use_generic = nullptr)
{
    if (use_generic) *use_generic = false;
    const fqnm_plan_desc& d = p->d;
    long long init[2] = {LLONG_MAX, LLONG_MIN};
    p->h_minmax[0] = init[0];
    p->h_minmax[1] = init[1];
    CUDA_TRY(cudaMemcpyAsync(p->d_minmax, p->h_minmax, 2 * sizeof(long long), cudaMemcpyHostToDevice, p->st));
    CUDA_TRY(launch_minmax(q, d.dtype, (int64_t)state_elems(d), p->d_minmax, p->st));
    p->launches++;
    CUDA_TRY(cudaMemcpyAsync(p->h_minmax + 2, p->d_minmax, 2 * sizeof(long long), cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaStreamSynchronize(p->st));
    long long mn = p->h_minmax[2], mx = p->h_minmax[3];
    const bool one_d = p->family == 2 || p->family == 3 || p->family == 4 || p->family == 6;
    if ((mn < p->lo || mx > p->hi) && use_generic && one_d && p->d8_lim > 0 && mn >= -p->d8_lim &&
        mx <= p->d8_lim) {
        *use_generic = true;            // inside the D8 range, beyond the fast closed form's domain
        return FQNM_OK;
    }
    if (mn < p->lo || mx > p->hi)
        return fail(FQNM_ERR_RANGE, "state range [%lld, %lld] outside the plan's admissible "
                    "range [%lld, %lld]", mn, mx, (long long)p->lo, (long long)p->hi);
    return FQNM_OK;
}

static int prof_begin(fqnm_plan_t* p)
{
    if (!p->prof) return FQNM_OK;
    if (p->ev_used + 2 > p->ev.size()) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            p->ev.push_back(e);
        }
    }
    CUDA_TRY(cudaEventRecord(p->ev[p->ev_used], p->st));
    return FQNM_OK;
}

static int prof_end(fqnm_plan_t* p)
{
    if (!p->prof) return FQNM_OK;
    CUDA_TRY(cudaEventRecord(p->ev[p->ev_used + 1], p->st));
    p->ev_used += 2;
    return FQNM_OK;
}

#define PROF_LAUNCH(expr)                                  \
    do {                                                   \
        int rc_ = prof_begin(p);                           \
        if (rc_ != FQNM_OK) return rc_;                    \
        CUDA_TRY(expr);                                    \
        if ((rc_ = prof_end(p)) != FQNM_OK) return rc_;    \
        p->launches++;                                     \
    } while (0)

// ---- 2D/3D range guard: the unsplit directional composition (Thm P:364-401)
// is not monotone in general once quantised (the per-direction increments of phi+ - phi-
// can add up past 1), so the maximum principle that keeps a 1D state inside the plan's
// admissible range [lo, hi] (where the fast closed-form maps are exact) is not available.
// The 2D/3D kernels compare every cell they store with [lo, hi] and set a device flag;
// the next launches return at once when it is set, and fqnm_step reports FQNM_ERR_RANGE
// after the loop (q unspecified then).  The multi-D range is clamped at plan time to
// |q| <= (2^31 - 1) / (1 + 4d), so the one step that leaves it cannot wrap int32.
static void md_guard_args(fqnm_plan_t* p, int** guard, int32_t* glo, int32_t* ghi)
{
    const bool on = p->md_guard && p->d.check_range;
    *guard = on ? p->md_guard : nullptr;
    *glo = (int32_t)(p->lo < INT32_MIN ? INT32_MIN : p->lo);
    *ghi = (int32_t)(p->hi > INT32_MAX ? INT32_MAX : p->hi);
}

static cudaError_t md_guard_reset(fqnm_plan_t* p)
{
    if (!p->md_guard || !p->d.check_range) return cudaSuccess;
    return cudaMemsetAsync(p->md_guard, 0, sizeof(int), p->st);
}


static int md_guard_result(fqnm_plan_t* p)
{
    if (!p->md_guard || !p->d.check_range) return FQNM_OK;
    CUDA_TRY(cudaMemcpyAsync(p->md_guard_host, p->md_guard, sizeof(int), cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaStreamSynchronize(p->st));
    if (*p->md_guard_host)
        return fail(FQNM_ERR_RANGE, "the 2D/3D state left the plan's admissible range [%lld, %lld] "
                    "during the call (the unsplit composition is not monotone); q is unspecified",
                    (long long)p->lo, (long long)p->hi);
    return FQNM_OK;
}

static int bmode_of(const fqnm_plan_desc& d)
{
    return d.boundary == FQNM_TRANSMISSIVE ? BM_TRANSMISSIVE
           : (d.boundary == FQNM_HALO ? BM_HALO : BM_PERIODIC);
}

#ifndef FQNM_K2S_GRID
#define FQNM_K2S_GRID (148 * 32)   // K2S grid cap in CTAs (windows are grid-strided over the warps)
#endif

static int launch_block(fqnm_plan_t* p, const int32_t* src, int32_t* dst, int ksteps)
{
    const fqnm_plan_desc& d = p->d;
    BlockedArgs a;
    std::memset(&a, 0, sizeof a);
    a.src = src;
    a.dst = dst;
    a.n = d.n_local;
    a.batch = d.batch;
    a.halo = d.boundary == FQNM_HALO ? d.halo : 0;
    a.ksteps = ksteps;
    a.KL = p->dep_left ? round4(ksteps) : 0;
    a.KR = p->dep_right ? round4(ksteps) : 0;
    a.bmode = bmode_of(d);
    a.guard = p->guard;
    // K2S geometry (V = 48): when the host proved the sign, or for the dual launch
    const bool sign_ok = d.boundary != FQNM_HALO && blocked_sign_has_rule(p->rule) && !p->no_sign &&
                         32 * BLOCKED_SIGN_V - a.KL - a.KR >= 4;
    if (sign_ok && (p->sign_hint || p->sign_dev)) {
        BlockedArgs b = a;
        // a one-signed state moves one way only: with every q >= 0 the transfer is
        // F_{j+1/2} = phi+(q_j) and a cell depends on its left neighbour alone (q <= 0: on
        // its right neighbour), so the window needs no halo on the other side
        const int sgn = p->sign_hint ? p->sign_hint : 1;
        if (sgn == 1) b.KR = 0; else b.KL = 0;
        const int64_t S2 = 32 * BLOCKED_SIGN_V - b.KL - b.KR;
        b.nwin = (d.n_local + S2 - 1) / S2;
        b.sign_bits = p->sign_hint ? nullptr : p->sign_dev;
        PROF_LAUNCH(launch_blocked_sign(p->rule, p->sign_hint ? p->sign_hint : 1, b, p->dr, p->st,
                                        FQNM_K2S_GRID));
        p->k2s_launches++;
        if (p->sign_hint) return FQNM_OK;
        a.sign_bits = p->sign_dev;                 // dual launch: the general K2 covers the rest
    }
    const int64_t S = 32 * p->V - a.KL - a.KR;
    if (S < 4) return fail(FQNM_ERR_ARG, "k = %d too large for V = %d", ksteps, p->V);
    a.nwin = (d.n_local + S - 1) / S;
    PROF_LAUNCH(launch_blocked(p->rule, p->V, p->minb, a, p->dr, p->st, 148 * 32));
    return FQNM_OK;
}

// K2P eligibility: one single-domain problem on the V = 32 / 2-CTA K2 variant with a rule
// the persistent kernel is built for; auto mode when a launch would have few waves of
// windows (the last partial wave of each launch is then a visible share of the time)
static bool use_persist(fqnm_plan_t* p, int64_t nb)
{
    const fqnm_plan_desc& d = p->d;
    if (p->persist == 0 || nb < 2) return false;
    if (p->family != 2 || d.batch != 1 || d.boundary == FQNM_HALO || p->V != 32 || p->minb != 2 ||
        !blocked_persist_has_rule(p->rule))
        return false;
    if (p->persist == 1) return true;
    const int64_t S = 32 * p->V - (p->dep_left ? round4(p->k) : 0) - (p->dep_right ? round4(p->k) : 0);
    const int64_t nwin = (d.n_local + S - 1) / S;
    // few waves of resident warps per launch: the last partial wave of every K2 launch is a
    // visible share (cfg3: 7.4 waves, K2P 6.35 vs K2 6.22 TCUPS); from ~48 waves on K2 wins
    // (EO 2^28: 3.89 vs 3.74; profiles/r02_tune_k2p.jsonl)
    return nwin < 16 * 148 * 16;
}

// sign: 0 voting kernel, 1 / 2 sign-specialised (K2PS); sign_bits: device sign bits of the
// input for the dual launch of the pipelined chunks (null: unconditional launch)
static int step_persist(fqnm_plan_t* p, void* q, int64_t nb, int64_t base, int64_t rem, int sign,
                        const int* sign_bits)
{
    const fqnm_plan_desc& d = p->d;
    const int kmax = (int)(base + (rem > 0 ? 1 : 0));
    PersistArgs a;
    std::memset(&a, 0, sizeof a);
    a.buf0 = (int32_t*)q;
    a.buf1 = (int32_t*)p->scratch;
    a.n = d.n_local;
    a.KL = p->dep_left ? round4(kmax) : 0;
    a.KR = p->dep_right ? round4(kmax) : 0;
    const int Vp = blocked_persist_V(p->rule, sign);
    if (sign == 1) a.KR = 0;            // one-signed state: one-sided dependence (see launch_block)
    else if (sign == 2) a.KL = 0;
    a.S = 32 * Vp - a.KL - a.KR;
    if (a.S < 4) return fail(FQNM_ERR_ARG, "k = %d too large for V = %d", kmax, Vp);
    a.nwin = (a.n + a.S - 1) / a.S;
    a.base = (int32_t)base;
    a.rem = (int32_t)rem;
    a.nblocks = (int32_t)nb;
    a.bmode = bmode_of(d);
    if (p->pflags_n < a.nwin) {
        if (p->pflags) cudaFree(p->pflags);
        p->pflags = nullptr;
        CUDA_TRY(cudaMalloc(&p->pflags, (size_t)a.nwin * sizeof(unsigned int)));
        CUDA_TRY(cudaMemsetAsync(p->pflags, 0, (size_t)a.nwin * sizeof(unsigned int), p->st));
        p->pflags_n = a.nwin;
        p->ptag = 1;
    }
    if (!p->pcounter) CUDA_TRY(cudaMalloc(&p->pcounter, sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(p->pcounter, 0, sizeof(unsigned long long), p->st));
    // flags carry tag_base + blocks completed; tags strictly increase across calls
    if (p->ptag > 0xF0000000u - (uint32_t)nb) {
        CUDA_TRY(cudaMemsetAsync(p->pflags, 0, (size_t)p->pflags_n * sizeof(unsigned int), p->st));
        p->ptag = 1;
    }
    a.flags = p->pflags;
    a.counter = p->pcounter;
    a.guard = p->guard;
    a.sign_bits = sign_bits;
    a.tag_base = p->ptag;
    p->ptag += (uint32_t)nb + 1;
    PROF_LAUNCH(launch_blocked_persist(p->rule, sign, a, p->dr, p->st));
    if (sign) p->k2s_launches++;
    return FQNM_OK;
}

static int halo_step_blocks(fqnm_plan_t* const* plans, int nplans, int64_t nsteps);

// A range-checked EO step whose state left the fast closed form's domain but stays within
// the D8 range (+-d8_lim): the same problem on a plan with the exact int64 rule, created
// on first use.  The maximum principle (Lemma P:210-212, under D8) keeps the state in
// [min q, max q] for the whole call, so one check decides the call.
static int step_generic_child(fqnm_plan_t* p, void* q, int64_t nsteps)
{
    if (!p->generic_child) {
        fqnm_plan_desc d = p->d;
        d.kappa_num = p->kap_num;
        d.kappa_den = p->kap_den;
        d.q_lo = -p->d8_lim;
        d.q_hi = p->d8_lim;
        d.check_range = 0;
        d.k = 0;
        d.stream = (void*)p->st;
        fqnm_plan_t* c = nullptr;
        const int rc = plan_build(&c, &d, true, /*trusted_range=*/true);
        if (rc != FQNM_OK) return rc;
        if (c->rule != R_GENERIC) { fqnm_destroy(c); return fail(FQNM_ERR_UNSUPPORTED, "no int64 fallback rule"); }
        p->generic_child = c;
    }
    fqnm_plan_t* c = p->generic_child;
    c->st = p->st;
    const int64_t l0 = c->launches;
    const int rc = fqnm_step(c, q, nsteps);
    p->launches += c->launches - l0;
    return rc;
}

extern "C" int fqnm_step(fqnm_plan_t* p, void* q, int64_t nsteps)
{
    if (p && p->d.boundary == FQNM_HALO && p->d.p2p) {
        if (nsteps < 0) return fail(FQNM_ERR_ARG, "nsteps must be >= 0");
        return halo_step_blocks(&p, 1, nsteps);
    }
    if (!p || !q) return fail(FQNM_ERR_ARG, "null argument");
    if (nsteps < 0) return fail(FQNM_ERR_ARG, "nsteps must be >= 0");
    if (!aligned16(q)) return fail(FQNM_ERR_ARG, "q must be 16-byte aligned");
    const fqnm_plan_desc& d = p->d;
    if (d.boundary == FQNM_HALO)
        return fail(FQNM_ERR_UNSUPPORTED, "split-domain plans step through fqnm_step_block");
    if (nsteps == 0) return FQNM_OK;
    int rc;
    p->sign_hint = p->sign_preset;
    if (d.check_range && d.nvar == 1) {
        bool gen = false;
        if ((rc = check_range(p, q, &gen)) != FQNM_OK) return rc;
        if (gen) return step_generic_child(p, q, nsteps);
        // the range check's min/max: a state of one sign keeps it for the call (D8
        // monotonicity, Lemma CFL), so K2 can run the sign-specialised K2S
        const long long mn = p->h_minmax[2], mx = p->h_minmax[3];
        if (p->family == 2 && blocked_sign_has_rule(p->rule))
            p->sign_hint = mn >= 0 ? 1 : (mx <= 0 ? 2 : 0);
    }
    const int bm = bmode_of(d);
    const int64_t n = d.n_local;
    const size_t bytes = state_elems(d) * elem_size(d);

    if (p->family == 3) {
        PROF_LAUNCH(launch_warp_ensemble(p->rule, p->V, (int32_t*)q, d.batch, nsteps, bm, p->dr, p->st));
        return FQNM_OK;
    }
    if (p->family == 4) {
        PROF_LAUNCH(launch_cta_ensemble(p->rule, (int32_t*)q, n, d.batch, nsteps, bm, p->dr, p->st));
        return FQNM_OK;
    }
    if (p->family == 6) {
        ResidentArgsHost h;
        int P, base, rem, H;
        if ((rc = resident_geometry(p, p->k, &P, &base, &rem, &H)) != FQNM_OK)
            return fail(rc, "resident stepper: invalid k = %d for n = %lld", p->k, (long long)n);
        if (P > p->res_P) return fail(FQNM_ERR_ARG, "resident stepper: edge buffers too small");
        h.src = (const int32_t*)q;
        h.dst = (int32_t*)p->scratch;
        h.edges = p->edges;
        h.flags = p->flags;
        h.tag_base = p->tag_base;
        h.n = n;
        h.nsteps = nsteps;
        h.P = P; h.base = base; h.rem = rem; h.H = H; h.k = p->k < H ? p->k : H;
        p->tag_base += (uint32_t)((nsteps + h.k - 1) / h.k) + 1;    // fresh tags for the next call
        h.bmode = bm;
        PROF_LAUNCH(launch_resident(p->rule, p->V, h, p->dr, p->st));
        CUDA_TRY(cudaMemcpyAsync(q, p->scratch, bytes, cudaMemcpyDeviceToDevice, p->st));
        return FQNM_OK;
    }
    // ping-pong families
    void* bufs[2] = {q, p->scratch};
    int cur = 0;
    if (p->family == 7 && p->stream2d) {
        Step2DArgs a;
        a.nx = p->nx;
        a.ny = p->ny;
        a.ksteps = (int32_t)step2d_stream_rows(p->nx, p->ny);
        a.bmode = bm;
        md_guard_args(p, &a.guard, &a.glo, &a.ghi);
        CUDA_TRY(md_guard_reset(p));
        for (int64_t s = 0; s < nsteps;) {
            a.src = (const int32_t*)bufs[cur];
            a.dst = (int32_t*)bufs[cur ^ 1];
            // two steps per launch (8192^2: EO 804 vs 629, linear 786 vs 666 GCUPS)
            if (p->k2s == 2 && s + 2 <= nsteps) {
                PROF_LAUNCH(launch_step2d_stream2(p->rule, p->same_xy, a, p->dr, p->dry, p->st));
                s += 2;
            } else {
                PROF_LAUNCH(launch_step2d_stream(p->rule, p->same_xy, a, p->dr, p->dry, p->st));
                s += 1;
            }
            cur ^= 1;
        }
        if (cur != 0) CUDA_TRY(cudaMemcpyAsync(q, bufs[cur], bytes, cudaMemcpyDeviceToDevice, p->st));
        return md_guard_result(p);
    }
    if (p->family == 7) {
        int64_t nb = (nsteps + p->k - 1) / p->k;
        if (nb % 2 == 1 && nsteps >= nb + 1) nb += 1;
        const int64_t base = nsteps / nb, rem = nsteps % nb;
        CUDA_TRY(md_guard_reset(p));
        for (int64_t b = 0; b < nb; ++b) {
            Step2DArgs a;
            a.src = (const int32_t*)bufs[cur];
            a.dst = (int32_t*)bufs[cur ^ 1];
            a.nx = p->nx;
            a.ny = p->ny;
            a.ksteps = (int)(base + (b < rem ? 1 : 0));
            a.bmode = bm;
            md_guard_args(p, &a.guard, &a.glo, &a.ghi);
            PROF_LAUNCH(launch_step2d(p->rule, p->same_xy, a, p->dr, p->dry, p->st));
            cur ^= 1;
        }
        if (cur != 0) CUDA_TRY(cudaMemcpyAsync(q, bufs[cur], bytes, cudaMemcpyDeviceToDevice, p->st));
        return md_guard_result(p);
    }
    if (p->family == 8) {
        Step3DArgs a;
        std::memset(&a, 0, sizeof a);
        a.nx = p->nx;
        a.ny = p->ny;
        a.nz = p->nz;
        a.zchunk = p->stream3d ? step3d_s_zchunk(p->nx, p->ny, p->nz) : step3d_zchunk(p->nx, p->ny, p->nz);
        a.bmode = bm;
        md_guard_args(p, &a.guard, &a.glo, &a.ghi);
        CUDA_TRY(md_guard_reset(p));
        for (int64_t s = 0; s < nsteps; ++s) {
            a.src = (const int32_t*)bufs[cur];
            a.dst = (int32_t*)bufs[cur ^ 1];
            if (p->stream3d)
                PROF_LAUNCH(launch_step3d_stream(p->rule, p->same_xy, a, p->dr, p->dry, p->drz, p->st));
            else
                PROF_LAUNCH(launch_step3d(p->rule, p->same_xy, a, p->dr, p->dry, p->drz, p->st));
            cur ^= 1;
        }
        if (cur != 0) CUDA_TRY(cudaMemcpyAsync(q, bufs[cur], bytes, cudaMemcpyDeviceToDevice, p->st));
        return md_guard_result(p);
    }
    if (p->family == 1 || p->family == 5) {
        for (int64_t s = 0; s < nsteps; ++s) {
            if (p->family == 1) {
                PROF_LAUNCH(launch_naive(p->rule, (const int32_t*)bufs[cur], (int32_t*)bufs[cur ^ 1], n,
                                         d.batch, bm, p->dr, p->st));
            } else {
                EulerArgs a;
                a.src = (const int64_t*)bufs[cur];
                a.dst = (int64_t*)bufs[cur ^ 1];
                a.n = n;
                a.batch = d.batch;
                a.nwin = (n + (32 * p->V - 2) - 1) / (32 * p->V - 2);
                a.delta = d.delta;
                a.s = p->s_e;
                a.g1 = p->g1_e;
                a.lam = d.dt_dx;
                a.mode = d.flux_kind == FQNM_EULER_ROE_DENSITY ? 1 : 0;
                a.bmode = bm;
                PROF_LAUNCH(launch_euler(p->V, a, p->st));
            }
            cur ^= 1;
        }
    } else {
        // temporally blocked: an even number of blocks so the result lands in q
        int64_t nb = (nsteps + p->k - 1) / p->k;
        if (nb % 2 == 1 && nsteps >= nb + 1) nb += 1;
        const int64_t base = nsteps / nb, rem = nsteps % nb;
        if (use_persist(p, nb)) {
            // K2PS when the range check proved the sign; for a pipelined chunk the sign is
            // known on the device only: K2PS (q >= 0) and the voting K2P are both launched and
            // the one the sign bits do not select returns at once
            const bool sign_rule = !p->no_sign && blocked_sign_has_rule(p->rule);
            const int sign = sign_rule ? p->sign_hint : 0;
            if (!sign && sign_rule && p->sign_dev) {
                if ((rc = step_persist(p, q, nb, base, rem, 1, p->sign_dev)) != FQNM_OK) return rc;
                if ((rc = step_persist(p, q, nb, base, rem, 0, p->sign_dev)) != FQNM_OK) return rc;
            } else if ((rc = step_persist(p, q, nb, base, rem, sign, nullptr)) != FQNM_OK) {
                return rc;
            }
            cur = (int)(nb & 1);
            if (cur != 0) CUDA_TRY(cudaMemcpyAsync(q, bufs[cur], bytes, cudaMemcpyDeviceToDevice, p->st));
            return FQNM_OK;
        }
        for (int64_t b = 0; b < nb; ++b) {
            int ks = (int)(base + (b < rem ? 1 : 0));
            if ((rc = launch_block(p, (const int32_t*)bufs[cur], (int32_t*)bufs[cur ^ 1], ks)) != FQNM_OK)
                return rc;
            cur ^= 1;
        }
    }
    if (cur != 0) CUDA_TRY(cudaMemcpyAsync(q, bufs[cur], bytes, cudaMemcpyDeviceToDevice, p->st));
    return FQNM_OK;
}

static void halo_args(fqnm_plan_t* p, BlockedArgs& a, int ksteps, uint32_t tag)
{
    const fqnm_plan_desc& d = p->d;
    std::memset(&a, 0, sizeof a);                       // every field defined (guard = null)
    a.src = (const int32_t*)p->hbuf[p->hcur];
    a.dst = (int32_t*)p->hbuf[p->hcur ^ 1];
    a.n = d.n_local;
    a.batch = 1;
    a.halo = d.halo;
    a.ksteps = ksteps;
    a.KL = p->dep_left ? round4(ksteps) : 0;
    a.KR = p->dep_right ? round4(ksteps) : 0;
    a.bmode = BM_HALO;
    const int64_t S = 32 * p->V - a.KL - a.KR;
    a.nwin = (d.n_local + S - 1) / S;
    a.p2p = 1;
    a.tag = tag;
    a.peer_left_dst = (int32_t*)p->lbuf[p->hcur ^ 1];
    a.peer_right_dst = (int32_t*)p->rbuf[p->hcur ^ 1];
    a.left_n = p->ln;
    a.right_n = p->rn;
    a.self_flags = p->hflags;
    a.peer_left_flags = p->lflags;
    a.peer_right_flags = p->rflags;
}

// Prime (every rank pushes the edges of its current buffer, tag t0), then the
// blocks: block b waits for t0 + b and pushes t0 + b + 1.  With several plans
// (virtual ranks on one device) the launches are interleaved rank by rank.
static int halo_step_blocks(fqnm_plan_t* const* plans, int nplans, int64_t nsteps)
{
    for (int i = 0; i < nplans; ++i) {
        fqnm_plan_t* p = plans[i];
        if (!p || !(p->d.boundary == FQNM_HALO && p->d.p2p))
            return fail(FQNM_ERR_ARG, "fqnm_step_group needs p2p split-domain plans");
        if (!p->hconnected) return fail(FQNM_ERR_ARG, "p2p plan not connected (fqnm_halo_connect)");
        if (p->d.n_local < 32 * p->V) return fail(FQNM_ERR_UNSUPPORTED, "p2p needs n_local >= one window");
    }
    if (nsteps == 0) return FQNM_OK;
    fqnm_plan_t* p0 = plans[0];
    const int k = p0->k;
    const int64_t nb = (nsteps + k - 1) / k;
    const uint32_t t0 = p0->htag;
    for (int i = 0; i < nplans; ++i) {
        fqnm_plan_t* p = plans[i];
        if (p->k != k || p->htag != t0) return fail(FQNM_ERR_ARG, "p2p plans out of step");
        BlockedArgs a;
        halo_args(p, a, k, t0);
        a.peer_left_dst = (int32_t*)p->lbuf[p->hcur];     // prime: neighbours' current buffers
        a.peer_right_dst = (int32_t*)p->rbuf[p->hcur];
        CUDA_TRY(launch_halo_prime(a, p->st));
        p->launches++;
    }
    int64_t done = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const int ks = (int)((nsteps - done) < k ? (nsteps - done) : k);
        for (int i = 0; i < nplans; ++i) {
            fqnm_plan_t* p = plans[i];
            BlockedArgs a;
            halo_args(p, a, ks, t0 + (uint32_t)b);
            PROF_LAUNCH(launch_blocked(p->rule, p->V, p->minb, a, p->dr, p->st, 148 * 32));
            p->hcur ^= 1;
        }
        done += ks;
    }
    for (int i = 0; i < nplans; ++i) plans[i]->htag = t0 + (uint32_t)nb + 1;
    return FQNM_OK;
}

extern "C" int fqnm_step_group(fqnm_plan_t* const* plans, int nplans, int64_t nsteps)
{
    if (!plans || nplans < 1) return fail(FQNM_ERR_ARG, "null argument");
    if (nsteps < 0) return fail(FQNM_ERR_ARG, "nsteps must be >= 0");
    return halo_step_blocks(plans, nplans, nsteps);
}

extern "C" int fqnm_halo_buffers(const fqnm_plan_t* p, void** buf0, void** buf1, unsigned int** flags)
{
    if (!p || !buf0 || !buf1 || !flags) return fail(FQNM_ERR_ARG, "null argument");
    if (!p->hbuf[0]) return fail(FQNM_ERR_ARG, "not a p2p split-domain plan");
    *buf0 = p->hbuf[0];
    *buf1 = p->hbuf[1];
    *flags = p->hflags;
    return FQNM_OK;
}

extern "C" int fqnm_halo_connect(fqnm_plan_t* p, void* left_buf0, void* left_buf1,
                                 unsigned int* left_flags, int64_t left_n, void* right_buf0,
                                 void* right_buf1, unsigned int* right_flags, int64_t right_n)
{
    if (!p || !left_buf0 || !left_buf1 || !left_flags || !right_buf0 || !right_buf1 || !right_flags)
        return fail(FQNM_ERR_ARG, "null argument");
    if (!p->hbuf[0]) return fail(FQNM_ERR_ARG, "not a p2p split-domain plan");
    if (left_n < p->d.halo || right_n < p->d.halo) return fail(FQNM_ERR_ARG, "neighbour smaller than the halo");
    p->lbuf[0] = left_buf0; p->lbuf[1] = left_buf1; p->lflags = left_flags; p->ln = left_n;
    p->rbuf[0] = right_buf0; p->rbuf[1] = right_buf1; p->rflags = right_flags; p->rn = right_n;
    p->hconnected = true;
    return FQNM_OK;
}

extern "C" int fqnm_halo_owned(const fqnm_plan_t* p, void** owned)
{
    if (!p || !owned) return fail(FQNM_ERR_ARG, "null argument");
    if (!p->hbuf[0]) return fail(FQNM_ERR_ARG, "not a p2p split-domain plan");
    *owned = (int32_t*)p->hbuf[p->hcur] + p->d.halo;
    return FQNM_OK;
}

extern "C" int fqnm_ipc_export(const void* dev_ptr, void* handle64)
{
    if (!dev_ptr || !handle64) return fail(FQNM_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    std::memcpy(handle64, &h, sizeof h);
    return FQNM_OK;
}

extern "C" int fqnm_ipc_open(const void* handle64, void** dev_ptr)
{
    if (!dev_ptr || !handle64) return fail(FQNM_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return FQNM_OK;
}

extern "C" int fqnm_ipc_close(void* dev_ptr)
{
    if (!dev_ptr) return fail(FQNM_ERR_ARG, "null argument");
    CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return FQNM_OK;
}

extern "C" int fqnm_step_block(fqnm_plan_t* p, const void* src, void* dst, int32_t ksteps)
{
    if (!p || !src || !dst) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.boundary != FQNM_HALO) return fail(FQNM_ERR_ARG, "fqnm_step_block needs a FQNM_HALO plan");
    if (src == dst) return fail(FQNM_ERR_ARG, "src and dst must differ");
    if (ksteps < 1 || ksteps > p->d.halo) return fail(FQNM_ERR_ARG, "need 1 <= ksteps <= halo");
    if (ksteps > max_block_steps(p, p->V)) return fail(FQNM_ERR_ARG, "ksteps too large for this plan");
    if (!aligned16(src) || !aligned16(dst)) return fail(FQNM_ERR_ARG, "buffers must be 16-byte aligned");
    return launch_block(p, (const int32_t*)src, (int32_t*)dst, ksteps);
}

extern "C" int fqnm_observe(const fqnm_plan_t* p, const void* q, double* u)
{
    if (!p || !q || !u) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.flux_kind == FQNM_EULER_ROE_DENSITY) {
        // density: u = delta q; momentum and energy are already float64 (bit copy)
        const int64_t n = p->d.n_local;
        for (int64_t b = 0; b < p->d.batch; ++b) {
            const int64_t* qb = (const int64_t*)q + b * 3 * n;
            double* ub = u + b * 3 * n;
            CUDA_TRY(launch_observe(qb, FQNM_I64, p->d.delta, ub, n, p->st));
            const_cast<fqnm_plan_t*>(p)->launches++;
            CUDA_TRY(cudaMemcpyAsync(ub + n, qb + n, 2 * n * sizeof(double),
                                     cudaMemcpyDeviceToDevice, p->st));
        }
        return FQNM_OK;
    }
    CUDA_TRY(launch_observe(q, p->d.dtype, p->d.delta, u, (int64_t)state_elems(p->d), p->st));
    const_cast<fqnm_plan_t*>(p)->launches++;
    return FQNM_OK;
}

// Pipelined end-to-end path for one large periodic scalar problem: the domain is cut
// into m chunks of C cells; chunk c is stepped independently on its extended region
// [cC - H, cC + C + H) (periodic wrap) as a transmissive problem, H >= nsteps, so its
// C inner cells are exact (their dependence cone, one cell per step and side, stays
// inside the region); the extra work is 2H/C.  Three device buffers rotate so that
// the H2D copy of chunk c+1 and the D2H copy of chunk c-1 overlap the stepping of
// chunk c (three streams, events).  The input range check of each extended region
// runs on the device and, if it fails, turns that chunk's launches into no-ops.
#ifndef FQNM_PIPE_RAMP
#define FQNM_PIPE_RAMP 1       // pipelined fqnm_step_host: ramped first/last chunks (C/8 .. C/2)
#endif
#ifndef FQNM_PIPE_PERSIST
#define FQNM_PIPE_PERSIST 1    // pipelined chunks step with K2P / K2PS
#endif
#ifndef FQNM_PIPE_DUAL
#define FQNM_PIPE_DUAL 0       // pipelined chunks: K2S + K2 dual launch on the device sign bits
                               // (measured slower on cfg4 e2e: 3535 vs 3602 GCUPS)
#endif
#ifndef FQNM_PIPE_SIGN_USE
#define FQNM_PIPE_SIGN_USE 1   // experiment switch: 0 = read the sign bits but keep K2
#endif
#ifndef FQNM_PIPE_SIGN
#define FQNM_PIPE_SIGN 0       // pipelined chunks: the host reads each chunk's sign bits and
                               // steps one-signed chunks with K2S (the per-chunk host wait
                               // measured 2977 vs 3615 GCUPS e2e; K2S on chunk-sized problems
                               // is not faster than the voting K2 either: dual 3539-3593)
#endif
#ifndef FQNM_PIPE_LOG2C
#define FQNM_PIPE_LOG2C 27     // largest chunk of the e2e pipeline: 2^27 cells
#endif
static int pipe_setup(fqnm_plan_t* p, int64_t nsteps)
{
    const int64_t n = p->d.n_local;
    const int64_t H = (nsteps + 31) / 32 * 32;
    int64_t m = 0, C = 0;
    for (int64_t mm = 4; mm <= 256; mm *= 2) {
        if (n % mm) break;
        const int64_t c = n / mm;
        if (c % 32) break;
        if (c <= ((int64_t)1 << FQNM_PIPE_LOG2C) && H * 16 <= c) { m = mm; C = c; break; }
    }
    if (!m) return FQNM_ERR_UNSUPPORTED;
    if (p->pipe_child && p->pipe_H == H && p->pipe_C == C) return FQNM_OK;
    pipe_release(p);
    // chunk list: m chunks of C, the first and last ramped when C/8 keeps the constraints
    const bool ramp = FQNM_PIPE_RAMP && m >= 3 && (C / 8) % 32 == 0 && H * 16 <= C / 8;
    {
        std::vector<int64_t> sz;
        if (ramp) { sz = {C / 8, C / 8, C / 4, C / 2}; }
        for (int64_t i = ramp ? 1 : 0; i < (ramp ? m - 1 : m); ++i) sz.push_back(C);
        if (ramp) { sz.push_back(C / 2); sz.push_back(C / 4); sz.push_back(C / 8); sz.push_back(C / 8); }
        int64_t st0 = 0;
        for (int64_t x : sz) { p->pipe_start.push_back(st0); p->pipe_size.push_back(x); st0 += x; }
        if (st0 != n) { pipe_release(p); return FQNM_ERR_UNSUPPORTED; }
    }
    for (int i = 0; i < (ramp ? 4 : 1); ++i) {
        fqnm_plan_desc d = p->d;
        d.n_local = d.n_global = (C >> i) + 2 * H;
        d.offset = 0;
        d.boundary = FQNM_TRANSMISSIVE;
        d.kappa_num = p->kap_num;
        d.kappa_den = p->kap_den;
        d.q_lo = p->lo;
        d.q_hi = p->hi;
        d.check_range = 0;
        d.k = p->k;
        d.stream = (void*)p->st;
        fqnm_plan_t* c = nullptr;
        int rc = plan_build(&c, &d, true);
        if (rc != FQNM_OK) { pipe_release(p); return rc; }
        if (c->family != 2 || c->rule != p->rule) {
            fqnm_destroy(c);
            pipe_release(p);
            return FQNM_ERR_UNSUPPORTED;
        }
        c->st = p->st;
        // chunks step with the persistent kernels (one launch for all blocks, no launch tails;
        // K2PS + voting K2P dual launch on the chunk's device sign bits): e2e 3.65 -> see
        // profiles/r02_tune_k2p.jsonl
        c->persist = FQNM_PIPE_PERSIST && blocked_persist_has_rule(c->rule) ? 1 : 0;
        p->pipe_kids[i] = c;
        if (i == 0) p->pipe_child = c;
    }
    m = (int64_t)p->pipe_size.size();
    p->pipe_H = H;
    p->pipe_C = C;
    p->pipe_m = m;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 3 && e == cudaSuccess; ++i) e = cudaMalloc(&p->pipe_buf[i], (size_t)(C + 2 * H) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&p->pipe_head, (size_t)H * 4);
    if (e == cudaSuccess) e = cudaMalloc(&p->pipe_guard, (size_t)m * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&p->pipe_sign, (size_t)m * sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&p->pipe_sign_host, (size_t)m * sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&p->pipe_guard_host, (size_t)m * sizeof(int));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->pipe_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->pipe_d2h, cudaStreamNonBlocking);
    for (int i = 0; i < 9 && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&p->pipe_ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        pipe_release(p);
        return fail(FQNM_ERR_NOMEM, "e2e pipeline buffers: %s", cudaGetErrorString(e));
    }
    p->pipe_guard_n = m;
    return FQNM_OK;
}

static int step_host_pipelined_impl(fqnm_plan_t* p, int32_t* qh, int64_t nsteps);

// on any failure, drain the three streams before returning so no copy into the caller's
// host buffer is still in flight
static int step_host_pipelined(fqnm_plan_t* p, int32_t* qh, int64_t nsteps)
{
    const int rc = step_host_pipelined_impl(p, qh, nsteps);
    if (rc != FQNM_OK) {
        cudaStreamSynchronize(p->pipe_h2d);
        cudaStreamSynchronize(p->st);
        cudaStreamSynchronize(p->pipe_d2h);
    }
    return rc;
}

// The host buffer is updated in place, so every read of q_host must precede the D2H that
// overwrites those cells:
//  * chunk c+1's left halo [(c+1)C - H, (c+1)C) is chunk c's output: H2D(c+1) is issued
//    before D2H(c) and D2H(c) waits on its event;
//  * the last chunk's right halo wraps to [0, H), chunk 0's output: it is copied into
//    pipe_head on the H2D stream before H2D(0) (so before D2H(0)) and taken from there;
//  * chunk c's right halo and chunk 0's left halo are outputs of later D2Hs, which follow
//    that chunk's H2D through the compute dependency.
static int step_host_pipelined_impl(fqnm_plan_t* p, int32_t* qh, int64_t nsteps)
{
    const int64_t n = p->d.n_local, C = p->pipe_C, H = p->pipe_H, m = p->pipe_m;
    auto kid_of = [&](int64_t c) -> fqnm_plan_t* {
        const int64_t sz = p->pipe_size[c];
        for (int i = 0; i < 4; ++i)
            if (p->pipe_kids[i] && (C >> i) == sz) return p->pipe_kids[i];
        return nullptr;
    };
    cudaEvent_t* ev_in = p->pipe_ev;
    cudaEvent_t* ev_comp = p->pipe_ev + 3;
    cudaEvent_t* ev_out = p->pipe_ev + 6;
    const bool check = p->d.check_range != 0;
    CUDA_TRY(cudaMemsetAsync(p->pipe_guard, 0, (size_t)m * sizeof(int), p->st));
    CUDA_TRY(cudaMemsetAsync(p->pipe_sign, 0, (size_t)m * sizeof(int), p->st));
    CUDA_TRY(cudaEventRecord(ev_comp[0], p->st));                 // guard reset before any use
    CUDA_TRY(cudaStreamWaitEvent(p->pipe_h2d, ev_comp[0], 0));
    CUDA_TRY(cudaMemcpyAsync(p->pipe_head, qh, (size_t)H * 4, cudaMemcpyHostToDevice, p->pipe_h2d));
    auto h2d = [&](int64_t c) -> int {
        const int b = (int)(c % 3);
        int32_t* buf = (int32_t*)p->pipe_buf[b];
        const int64_t E = p->pipe_size[c] + 2 * H;
        if (c >= 3) CUDA_TRY(cudaStreamWaitEvent(p->pipe_h2d, ev_out[b], 0));   // buffer free
        int64_t s0 = p->pipe_start[c] - H;
        if (s0 < 0) s0 += n;
        const int64_t first = (s0 + E <= n) ? E : n - s0;
        CUDA_TRY(cudaMemcpyAsync(buf, qh + s0, (size_t)first * 4, cudaMemcpyHostToDevice, p->pipe_h2d));
        if (first < E) {
            // wrapped part: [0, E - first) of the domain; its first H cells may already be
            // chunk 0's output in q_host, so they come from the saved head
            const int64_t w = E - first, wh = w < H ? w : H;
            CUDA_TRY(cudaMemcpyAsync(buf + first, p->pipe_head, (size_t)wh * 4, cudaMemcpyDeviceToDevice,
                                     p->pipe_h2d));
            if (w > wh)
                CUDA_TRY(cudaMemcpyAsync(buf + first + wh, qh + wh, (size_t)(w - wh) * 4,
                                         cudaMemcpyHostToDevice, p->pipe_h2d));
        }
        CUDA_TRY(cudaEventRecord(ev_in[b], p->pipe_h2d));
        return FQNM_OK;
    };
    int rc = h2d(0);
    if (rc != FQNM_OK) return rc;
    for (int64_t c = 0; c < m; ++c) {
        const int b = (int)(c % 3);
        int32_t* buf = (int32_t*)p->pipe_buf[b];
        const int64_t Cc = p->pipe_size[c], E = Cc + 2 * H;
        fqnm_plan_t* ch = kid_of(c);
        if (!ch) return fail(FQNM_ERR_ARG, "e2e pipeline: no child plan for chunk %lld", (long long)c);
        ch->st = p->st;                                            // the caller's current stream
        if (c + 1 < m && (rc = h2d(c + 1)) != FQNM_OK) return rc;  // reads chunk c's cells: first
        // range check + stepping on the compute stream
        CUDA_TRY(cudaStreamWaitEvent(p->st, ev_in[b], 0));
        if (check) {
            // range guard of the extended chunk + its sign bits (K2S / K2 dual launch)
            CUDA_TRY(launch_range_sign_guard(buf, E, p->lo, p->hi, p->pipe_guard + c,
                                             p->pipe_sign + c, p->st));
            p->launches++;
            ch->guard = p->pipe_guard + c;
            ch->sign_dev = (FQNM_PIPE_DUAL || ch->persist == 1) ? p->pipe_sign + c : nullptr;
            if (!FQNM_PIPE_DUAL && FQNM_PIPE_SIGN && blocked_sign_has_rule(ch->rule)) {
                // read the chunk's sign bits on the host (measured slower, off by default)
                CUDA_TRY(cudaMemcpyAsync(p->pipe_sign_host + c, p->pipe_sign + c, sizeof(int),
                                         cudaMemcpyDeviceToHost, p->st));
                CUDA_TRY(cudaStreamSynchronize(p->st));
                const int bits = p->pipe_sign_host[c];
                ch->sign_preset = !FQNM_PIPE_SIGN_USE ? 0 : (bits & 1) == 0 ? 1 : ((bits & 2) == 0 ? 2 : 0);
            }
        } else {
            ch->guard = nullptr;
            ch->sign_dev = nullptr;
        }
        const int64_t l0 = ch->launches;
        rc = fqnm_step(ch, buf, nsteps);
        p->launches += ch->launches - l0;
        ch->guard = nullptr;
        ch->sign_dev = nullptr;
        ch->sign_preset = 0;
        if (rc != FQNM_OK) return rc;
        CUDA_TRY(cudaEventRecord(ev_comp[b], p->st));
        // D2H of the inner cells, after the stepping and after H2D(c+1) read their tail
        CUDA_TRY(cudaStreamWaitEvent(p->pipe_d2h, ev_comp[b], 0));
        if (c + 1 < m) CUDA_TRY(cudaStreamWaitEvent(p->pipe_d2h, ev_in[(c + 1) % 3], 0));
        CUDA_TRY(cudaMemcpyAsync(qh + p->pipe_start[c], buf + H, (size_t)Cc * 4, cudaMemcpyDeviceToHost,
                                 p->pipe_d2h));
        CUDA_TRY(cudaEventRecord(ev_out[b], p->pipe_d2h));
    }
    if (check)
        CUDA_TRY(cudaMemcpyAsync(p->pipe_guard_host, p->pipe_guard, (size_t)m * sizeof(int),
                                 cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaStreamSynchronize(p->st));
    CUDA_TRY(cudaStreamSynchronize(p->pipe_d2h));
    if (check)
        for (int64_t c = 0; c < m; ++c)
            if (p->pipe_guard_host[c])
                return fail(FQNM_ERR_RANGE, "state outside the plan's admissible range [%lld, %lld] "
                            "in chunk %lld (q_host is partially stepped)", (long long)p->lo,
                            (long long)p->hi, (long long)c);
    return FQNM_OK;
}

// fqnm_step_host on an ensemble (warp / CTA ensemble kernels, independent problems): the batch
// is cut into up to 16 chunks of whole problems; chunk c's H2D copy, stepping and D2H copy run
// on three streams, so the copies of neighbouring chunks overlap the stepping (no halos, no
// buffer rotation: every chunk has its own region of the device buffer).  Same result as
// the plain path (the kernels step problems independently).
static int step_host_ensemble(fqnm_plan_t* p, int32_t* qh, int64_t nsteps)
{
    const fqnm_plan_desc& d = p->d;
    const int64_t n = d.n_local, B = d.batch;
    const int m = (int)(B < 16 ? B : 16);
    cudaError_t e = cudaSuccess;
    if (!p->ens_h2d) {
        e = cudaStreamCreateWithFlags(&p->ens_h2d, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->ens_d2h, cudaStreamNonBlocking);
        for (int i = 0; i < 33 && e == cudaSuccess; ++i)
            e = cudaEventCreateWithFlags(&p->ens_ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(FQNM_ERR_CUDA, "ensemble e2e streams: %s", cudaGetErrorString(e));
    }
    int32_t* dev = (int32_t*)p->e2e_dev;
    const int bm = bmode_of(d);
    int rc = FQNM_OK;
    // the caller's stream orders this call after its earlier work: the copies start after it
    e = cudaEventRecord(p->ens_ev[32], p->st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->ens_h2d, p->ens_ev[32], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->ens_d2h, p->ens_ev[32], 0);
    for (int c = 0; c < m && e == cudaSuccess; ++c) {
        const int64_t b0 = B * c / m, b1 = B * (c + 1) / m;
        const size_t off = (size_t)b0 * n, cnt = (size_t)(b1 - b0) * n;
        e = cudaMemcpyAsync(dev + off, qh + off, cnt * 4, cudaMemcpyHostToDevice, p->ens_h2d);
        if (e == cudaSuccess) e = cudaEventRecord(p->ens_ev[2 * c], p->ens_h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->st, p->ens_ev[2 * c], 0);
        if (e != cudaSuccess) break;
        if (p->family == 3)
            e = launch_warp_ensemble(p->rule, p->V, dev + off, b1 - b0, nsteps, bm, p->dr, p->st);
        else
            e = launch_cta_ensemble(p->rule, dev + off, n, b1 - b0, nsteps, bm, p->dr, p->st);
        p->launches++;
        if (e == cudaSuccess) e = cudaEventRecord(p->ens_ev[2 * c + 1], p->st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->ens_d2h, p->ens_ev[2 * c + 1], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(qh + off, dev + off, cnt * 4, cudaMemcpyDeviceToHost, p->ens_d2h);
    }
    // drain all three streams before returning, also on failure (no copy into the caller's
    // buffer may still be in flight)
    cudaError_t e2 = cudaStreamSynchronize(p->ens_h2d);
    cudaError_t e3 = cudaStreamSynchronize(p->st);
    cudaError_t e4 = cudaStreamSynchronize(p->ens_d2h);
    if (e == cudaSuccess) e = e2 != cudaSuccess ? e2 : (e3 != cudaSuccess ? e3 : e4);
    if (e != cudaSuccess) rc = fail(FQNM_ERR_CUDA, "ensemble e2e pipeline: %s", cudaGetErrorString(e));
    return rc;
}

extern "C" int fqnm_step_host(fqnm_plan_t* p, void* q_host, int64_t nsteps)
{
    if (!p || !q_host) return fail(FQNM_ERR_ARG, "null argument");
    if (nsteps < 0) return fail(FQNM_ERR_ARG, "nsteps must be >= 0");
    const fqnm_plan_desc& d = p->d;
    if (nsteps > 0 && d.nvar == 1 && d.batch == 1 && d.boundary == FQNM_PERIODIC && p->family == 2 &&
        d.n_local >= ((int64_t)1 << 24) && pipe_setup(p, nsteps) == FQNM_OK)
        return step_host_pipelined(p, (int32_t*)q_host, nsteps);
    const size_t bytes = state_elems(p->d) * elem_size(p->d);
    if (!p->e2e_dev) {
        cudaError_t e = cudaMalloc(&p->e2e_dev, bytes);
        if (e != cudaSuccess) return fail(FQNM_ERR_NOMEM, "cudaMalloc e2e: %s", cudaGetErrorString(e));
        p->e2e_bytes = bytes;
    }
    // ensembles without the (whole-buffer, synchronous) range check: chunked pipeline
    if (nsteps > 0 && d.nvar == 1 && d.batch >= 4 && (p->family == 3 || p->family == 4) &&
        !d.check_range && bytes >= ((size_t)1 << 22))
        return step_host_ensemble(p, (int32_t*)q_host, nsteps);
    CUDA_TRY(cudaMemcpyAsync(p->e2e_dev, q_host, bytes, cudaMemcpyHostToDevice, p->st));
    int rc = fqnm_step(p, p->e2e_dev, nsteps);
    if (rc != FQNM_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(q_host, p->e2e_dev, bytes, cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaStreamSynchronize(p->st));
    return FQNM_OK;
}

// ---- level-space diagnostics ----------------------------------------------
struct DevScratch {                       // small RAII bundle for the synchronous diagnostics
    std::vector<void*> ptrs;
    ~DevScratch() { for (void* x : ptrs) cudaFree(x); }
    template <typename T> cudaError_t alloc(T** out, size_t count)
    {
        cudaError_t e = cudaMalloc((void**)out, count * sizeof(T));
        if (e == cudaSuccess) ptrs.push_back(*out);
        return e;
    }
};

// The level channel: the whole state of a scalar plan (one contiguous segment),
// the density component (var 0) of each problem of an Euler plan.
struct LevelSegments {
    int64_t count, len, stride;   // elements
};
static LevelSegments level_segments(const fqnm_plan_desc& d)
{
    if (d.nvar == 1) return {1, (int64_t)state_elems(d), 0};
    return {d.batch, d.n_local, (int64_t)d.nvar * d.n_local};
}
static const void* seg_ptr(const fqnm_plan_t* p, const void* q, int64_t s, int64_t stride)
{
    return (const char*)q + (size_t)(s * stride) * elem_size(p->d);
}

static int levels_impl(const fqnm_plan_t* p, const void* q, int64_t lo, int64_t L,
                       unsigned int* counts, fqnm_level_stats* out)
{
    const LevelSegments sg = level_segments(p->d);
    const int64_t n = sg.count * sg.len;
    DevScratch sc;
    unsigned long long* dull = nullptr;     // [0] outside, [1] occupied
    double* dacc = nullptr;
    CUDA_TRY(sc.alloc(&dull, 2));
    CUDA_TRY(sc.alloc(&dacc, 1));
    CUDA_TRY(cudaMemsetAsync(dull, 0, 2 * sizeof(unsigned long long), p->st));
    CUDA_TRY(cudaMemsetAsync(dacc, 0, sizeof(double), p->st));
    CUDA_TRY(cudaMemsetAsync(counts, 0, (size_t)L * sizeof(unsigned int), p->st));
    for (int64_t b = 0; b < sg.count; ++b)
        CUDA_TRY(launch_histogram(seg_ptr(p, q, b, sg.stride), p->d.dtype, sg.len, lo, L, counts, dull,
                                  p->st));
    CUDA_TRY(launch_clogc(counts, L, dacc, dull + 1, p->st));
    unsigned long long h[2];
    double acc;
    CUDA_TRY(cudaMemcpyAsync(h, dull, sizeof h, cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaMemcpyAsync(&acc, dacc, sizeof acc, cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaStreamSynchronize(p->st));
    const double N = (double)(n - (int64_t)h[0]);
    out->outside = (int64_t)h[0];
    out->occupied = (int64_t)h[1];
    out->S = N > 0 ? std::log(N) - acc / N : 0.0;     // -sum (c/N) log(c/N)
    out->N_eff = std::exp(out->S);
    return FQNM_OK;
}

extern "C" int fqnm_levels(const fqnm_plan_t* p, const void* q, int64_t lo, int64_t hi,
                           uint32_t* counts_dev, fqnm_level_stats* out)
{
    if (!p || !q || !out) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.boundary == FQNM_HALO)
        return fail(FQNM_ERR_UNSUPPORTED, "level diagnostics: non-halo plans only");
    if (hi < lo || hi - lo > ((int64_t)1 << 30)) return fail(FQNM_ERR_ARG, "need lo <= hi, hi - lo <= 2^30");
    const int64_t L = hi - lo + 1;
    DevScratch sc;
    unsigned int* counts = counts_dev;
    if (!counts) CUDA_TRY(sc.alloc(&counts, (size_t)L));
    return levels_impl(p, q, lo, L, counts, out);
}

extern "C" int fqnm_transitions(const fqnm_plan_t* p, const void* q0, const void* q1, int64_t lo,
                                int64_t hi, fqnm_transition_stats* out)
{
    if (!p || !q0 || !q1 || !out) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.boundary == FQNM_HALO)
        return fail(FQNM_ERR_UNSUPPORTED, "level diagnostics: non-halo plans only");
    if (hi < lo || hi - lo > ((int64_t)1 << 30)) return fail(FQNM_ERR_ARG, "need lo <= hi, hi - lo <= 2^30");
    const int64_t L = hi - lo + 1;
    const LevelSegments sg = level_segments(p->d);
    const int64_t n = sg.count * sg.len;
    DevScratch sc;
    unsigned int *c0 = nullptr, *c1 = nullptr, *vals = nullptr;
    unsigned long long *keys = nullptr, *dull = nullptr;   // dull: [0] overflow [1] npairs [2] maxbits
    double* rowsum = nullptr;
    unsigned long long cap = 1024;
    while (cap < 2ull * (unsigned long long)n) cap <<= 1;
    CUDA_TRY(sc.alloc(&c0, (size_t)L));
    CUDA_TRY(sc.alloc(&c1, (size_t)L));
    CUDA_TRY(sc.alloc(&keys, cap));
    CUDA_TRY(sc.alloc(&vals, cap));
    CUDA_TRY(sc.alloc(&rowsum, (size_t)L));
    CUDA_TRY(sc.alloc(&dull, 3));
    int rc;
    if ((rc = levels_impl(p, q0, lo, L, c0, &out->before)) != FQNM_OK) return rc;
    if ((rc = levels_impl(p, q1, lo, L, c1, &out->after)) != FQNM_OK) return rc;
    CUDA_TRY(cudaMemsetAsync(keys, 0xff, cap * sizeof(unsigned long long), p->st));
    CUDA_TRY(cudaMemsetAsync(vals, 0, cap * sizeof(unsigned int), p->st));
    CUDA_TRY(cudaMemsetAsync(rowsum, 0, (size_t)L * sizeof(double), p->st));
    CUDA_TRY(cudaMemsetAsync(dull, 0, 3 * sizeof(unsigned long long), p->st));
    for (int64_t b = 0; b < sg.count; ++b)
        CUDA_TRY(launch_pairs(seg_ptr(p, q0, b, sg.stride), seg_ptr(p, q1, b, sg.stride), p->d.dtype,
                              sg.len, lo, L, keys, vals, cap, dull, p->st));
    CUDA_TRY(launch_rowsums(keys, vals, cap, L, c0, rowsum, dull + 1, p->st));
    CUDA_TRY(launch_defect(rowsum, c0, c1, L, dull + 2, p->st));
    unsigned long long h[3];
    CUDA_TRY(cudaMemcpyAsync(h, dull, sizeof h, cudaMemcpyDeviceToHost, p->st));
    CUDA_TRY(cudaStreamSynchronize(p->st));
    out->overflow = (int64_t)h[0];
    out->nonzeros = (int64_t)h[1];
    double rho;
    std::memcpy(&rho, &h[2], sizeof rho);
    out->rho = rho;
    out->dS = out->after.S - out->before.S;
    return FQNM_OK;
}

extern "C" int fqnm_get_info(const fqnm_plan_t* p, fqnm_plan_info* info)
{
    if (!p || !info) return fail(FQNM_ERR_ARG, "null argument");
    fill_info(p, info);
    return FQNM_OK;
}

extern "C" int fqnm_transfer(const fqnm_plan_t* p, int64_t q, int64_t* phi_plus, int64_t* phi_minus)
{
    if (!p || !phi_plus || !phi_minus) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.nvar != 1) return fail(FQNM_ERR_ARG, "scalar plans only");
    if (p->rule == R_TWOPOINT || p->rule == R_TP_FAST)
        return fail(FQNM_ERR_UNSUPPORTED, "two-point rule has no split maps: use fqnm_transfer2");
    *phi_plus = host_phi(p->hp, q, p->d.rounding);
    *phi_minus = host_phi(p->hm, q, p->d.rounding);
    return FQNM_OK;
}

extern "C" int fqnm_transfer_device(const fqnm_plan_t* p, const int32_t* q, int32_t* pp, int32_t* pm,
                                    int64_t n)
{
    if (!p || !q || !pp || !pm) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.nvar != 1) return fail(FQNM_ERR_ARG, "scalar plans only");
    if (n <= 0) return FQNM_OK;
    CUDA_TRY(launch_transfer(p->rule, q, pp, pm, n, p->dr, p->st));
    const_cast<fqnm_plan_t*>(p)->launches++;
    return FQNM_OK;
}

static int64_t host_transfer2(const fqnm_plan_t* p, int64_t qL, int64_t qR)
{
    const int rd = p->d.rounding;
    if (p->rule != R_TWOPOINT && p->rule != R_TP_FAST) return host_phi(p->hp, qL, rd) + host_phi(p->hm, qR, rd);
    const DevRule& r = p->dr;
    const i128 L = qL, R = qR;
    i128 num;
    if (r.tp_kind == FQNM_BURGERS_LF2) {
        num = (i128)r.tp_c2 * (L * L + R * R) + (i128)r.tp_c1 * (L - R);
    } else {
        const i128 a = L > 0 ? L : 0, b = R < 0 ? R : 0;
        num = (i128)r.tp_c2 * (r.tp_kind == FQNM_BURGERS_GODUNOV ? (a * a > b * b ? a * a : b * b)
                                                                : a * a + b * b);
    }
    return (int64_t)round128(num, r.tp_den, rd);
}

extern "C" int fqnm_transfer2(const fqnm_plan_t* p, int64_t qL, int64_t qR, int64_t* T)
{
    if (!p || !T) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.nvar != 1 || p->family >= 7) return fail(FQNM_ERR_ARG, "1D scalar plans only");
    *T = host_transfer2(p, qL, qR);
    return FQNM_OK;
}

extern "C" int fqnm_transfer2_device(const fqnm_plan_t* p, const int32_t* qL, const int32_t* qR,
                                     int32_t* T, int64_t n)
{
    if (!p || !qL || !qR || !T) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.nvar != 1 || p->family >= 7) return fail(FQNM_ERR_ARG, "1D scalar plans only");
    if (n <= 0) return FQNM_OK;
    CUDA_TRY(launch_transfer2(p->rule, qL, qR, T, n, p->dr, p->st));
    const_cast<fqnm_plan_t*>(p)->launches++;
    return FQNM_OK;
}

extern "C" int fqnm_equivalence(fqnm_plan_t* a, const fqnm_plan_t* b, void* q, int64_t nsteps,
                                int64_t pair_capacity, fqnm_equivalence_stats* out)
{
    if (!a || !b || !q || !out) return fail(FQNM_ERR_ARG, "null argument");
    if (nsteps < 0 || pair_capacity < 0) return fail(FQNM_ERR_ARG, "nsteps and pair_capacity must be >= 0");
    const fqnm_plan_desc &da = a->d, &db = b->d;
    if (da.nvar != 1 || db.nvar != 1 || a->family >= 7 || b->family >= 7)
        return fail(FQNM_ERR_ARG, "equivalence needs 1D scalar plans");
    if (da.batch != 1 || db.batch != 1 || da.boundary == FQNM_HALO || db.boundary == FQNM_HALO)
        return fail(FQNM_ERR_ARG, "equivalence needs single, unsplit problems");
    if (da.n_local != db.n_local || da.boundary != db.boundary)
        return fail(FQNM_ERR_ARG, "plans differ in N or boundary");
    if (((uintptr_t)q & 3) != 0) return fail(FQNM_ERR_ARG, "q must be 4-byte aligned");
    const int64_t n = da.n_local;
    const int bm = da.boundary == FQNM_PERIODIC ? BM_PERIODIC : BM_TRANSMISSIVE;
    std::memset(out, 0, sizeof *out);
    // pair table over the union of the two plans' ranges
    const int64_t lo = a->lo < b->lo ? a->lo : b->lo, hi = a->hi > b->hi ? a->hi : b->hi;
    const int64_t L = hi - lo + 1;
    unsigned long long cap = 0;
    if (pair_capacity > 0) {
        if (L >= ((int64_t)1 << 31)) return fail(FQNM_ERR_ARG, "range too wide for pair tracking");
        cap = 1;
        while ((int64_t)cap < pair_capacity) cap <<= 1;
    }
    int32_t *buf = nullptr, *T = nullptr;
    unsigned long long *counters = nullptr, *keys = nullptr, *cnt2 = nullptr;
    unsigned int* vals = nullptr;
    int rc = FQNM_OK;
    cudaError_t e = cudaSuccess;
    const unsigned long long init[3] = {0ull, ~0ull, 0ull};
    unsigned long long hc[3] = {0, 0, 0}, h2[2] = {0, 0};
    cudaStream_t st = a->st;
    auto ok = [&](cudaError_t x) { if (x != cudaSuccess && e == cudaSuccess) e = x; return e == cudaSuccess; };
    if (ok(cudaMalloc(&buf, (size_t)n * 4)) && ok(cudaMalloc(&T, (size_t)(n + 1) * 4)) &&
        ok(cudaMalloc(&counters, 3 * sizeof(unsigned long long))) &&
        ok(cudaMalloc(&cnt2, 2 * sizeof(unsigned long long))) &&
        ok(cudaMemcpyAsync(counters, init, sizeof init, cudaMemcpyHostToDevice, st)) &&
        ok(cudaMemsetAsync(cnt2, 0, 2 * sizeof(unsigned long long), st))) {
        if (cap) {
            if (ok(cudaMalloc(&keys, cap * sizeof(unsigned long long))) &&
                ok(cudaMalloc(&vals, cap * sizeof(unsigned int)))) {
                ok(cudaMemsetAsync(keys, 0xff, cap * sizeof(unsigned long long), st));
                ok(cudaMemsetAsync(vals, 0, cap * sizeof(unsigned int), st));
            }
        }
        int32_t* cur = (int32_t*)q;
        int32_t* nxt = buf;
        for (int64_t s = 0; s < nsteps && e == cudaSuccess; ++s) {
            ok(launch_equiv_step(cur, nxt, T, n, bm, a->dr, a->rule, b->dr, b->rule, s, counters,
                                 keys, vals, cap ? cap - 1 : 0, lo, L, st));
            a->launches += 2;
            int32_t* t = cur; cur = nxt; nxt = t;
        }
        if (e == cudaSuccess && cur != (int32_t*)q)
            ok(cudaMemcpyAsync(q, cur, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
        if (e == cudaSuccess && cap) ok(launch_equiv_count(keys, vals, cap, cnt2, st));
        if (e == cudaSuccess) ok(cudaMemcpyAsync(hc, counters, sizeof hc, cudaMemcpyDeviceToHost, st));
        if (e == cudaSuccess) ok(cudaMemcpyAsync(h2, cnt2, sizeof h2, cudaMemcpyDeviceToHost, st));
        if (e == cudaSuccess) ok(cudaStreamSynchronize(st));
    }
    cudaFree(buf); cudaFree(T); cudaFree(counters); cudaFree(cnt2); cudaFree(keys); cudaFree(vals);
    if (e != cudaSuccess) return fail(FQNM_ERR_CUDA, "equivalence: %s", cudaGetErrorString(e));
    const int64_t nI = bm == BM_PERIODIC ? n : n + 1;
    out->interface_evals = nsteps * nI;
    out->mismatches = (int64_t)hc[0];
    out->first_mismatch_step = hc[1] == ~0ull ? -1 : (int64_t)hc[1];
    out->overflow = (int64_t)hc[2];
    out->visited_pairs = cap ? (int64_t)h2[0] : -1;
    out->mismatched_pairs = cap ? (int64_t)h2[1] : -1;
    return rc;
}

extern "C" int fqnm_roe_transfer_device(const fqnm_plan_t* p, const int64_t* qL, const int64_t* qR,
                                        int64_t* T, int64_t n)
{
    if (!p || !qL || !qR || !T) return fail(FQNM_ERR_ARG, "null argument");
    if (p->d.nvar != 3) return fail(FQNM_ERR_ARG, "Euler plans only");
    if (n <= 0) return FQNM_OK;
    CUDA_TRY(launch_roe_transfer(qL, qR, T, n, p->d.delta, p->s_e, p->g1_e, p->st));
    const_cast<fqnm_plan_t*>(p)->launches++;
    return FQNM_OK;
}

static void fill_info(const fqnm_plan_t* p, fqnm_plan_info* info)
{
    std::memset(info, 0, sizeof *info);
    info->kappa_num = p->kap_num;
    info->kappa_den = p->kap_den;
    info->q_lo = p->lo;
    info->q_hi = p->hi;
    info->rule = p->rule;
    info->k = p->k;
    info->cells_per_thread = p->V;
    info->kernel = p->family;
    info->scratch_bytes = (int64_t)p->scratch_bytes;
    info->s_euler = p->s_e;
    info->g1_euler = p->g1_e;
    info->d8_lim = p->d8_lim;
    info->k2s_launches = p->k2s_launches;
}

extern "C" int fqnm_plan_validate(const fqnm_plan_desc* d, fqnm_plan_info* info)
{
    if (!d || !info) return fail(FQNM_ERR_ARG, "null argument");
    fqnm_plan_t* p = nullptr;
    int rc = plan_build(&p, d, /*allocate=*/false);
    if (rc != FQNM_OK) return rc;
    fill_info(p, info);
    delete p;
    return FQNM_OK;
}

extern "C" int fqnm_profile_enable(fqnm_plan_t* p, int enable)
{
    if (!p) return fail(FQNM_ERR_ARG, "null plan");
    p->prof = enable != 0;
    return FQNM_OK;
}

extern "C" int fqnm_profile_read(fqnm_plan_t* p, double* total_ms, int64_t* launches)
{
    if (!p || !total_ms || !launches) return fail(FQNM_ERR_ARG, "null argument");
    CUDA_TRY(cudaStreamSynchronize(p->st));
    double tot = 0;
    for (size_t i = 0; i + 1 < p->ev_used; i += 2) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]));
        tot += ms;
    }
    *total_ms = tot;
    *launches = (int64_t)(p->ev_used / 2);
    p->ev_used = 0;
    return FQNM_OK;
}

extern "C" int fqnm_debug_override(fqnm_plan_t* p, int32_t kernel, int32_t k, int32_t V)
{
    if (!p) return fail(FQNM_ERR_ARG, "null plan");
    const fqnm_plan_desc& d = p->d;
    if (d.nvar == 3) {
        if (V && !euler_has_V(V)) return fail(FQNM_ERR_UNSUPPORTED, "Euler V must be 1, 2 or 4");
        if (V) p->V = V;
        return FQNM_OK;
    }
    if (p->family == 8) {                 // 3D: kernel 8 = K8 CTA tiles, 10 = K10 warp streaming
        if (k || V || (kernel && kernel != 8 && kernel != 10))
            return fail(FQNM_ERR_UNSUPPORTED, "3D plans: kernel 8 or 10, one step per launch");
        if (kernel) p->stream3d = kernel == 10;
        return FQNM_OK;
    }
    if (p->family == 7) {                 // 2D: kernel 7 = K7 smem-tiled (k <= 4), 9 = K9 streaming (k <= 2)
        if (kernel == 9) p->stream2d = true;
        else if (kernel == 7) p->stream2d = false;
        else if (kernel) return fail(FQNM_ERR_UNSUPPORTED, "2D plans: kernel 7 or 9");
        if (k) {
            if (p->stream2d) {
                if (k > 2) return fail(FQNM_ERR_ARG, "K9: k = 1 or 2");
                p->k2s = k;
            } else {
                if (k > STEP2D_KMAX) return fail(FQNM_ERR_ARG, "2D plans: k <= %d", STEP2D_KMAX);
                p->k = k;
            }
        }
        return FQNM_OK;
    }
    bool allow_sign = false;
    if (kernel == 22) {                 // K2, with K2S where the range check proves a sign
        kernel = 2;
        allow_sign = true;
    }
    if (kernel >= 100) {               // K2 with a register-cap variant: 2 + 100 * minb
        p->minb = kernel / 100;
        kernel = kernel % 100;
    }
    bool persist_sign = false;
    if (kernel == 32) {                 // K2P, with the sign-specialised K2PS where proved
        kernel = 12;
        persist_sign = true;
    }
    if (kernel == 12) {                 // K2P persistent stepper (K2 geometry V = 32, 2 CTAs/SM)
        if (d.nvar != 1 || p->family >= 7 || d.batch != 1 || d.boundary == FQNM_HALO ||
            !blocked_persist_has_rule(p->rule))
            return fail(FQNM_ERR_UNSUPPORTED, "K2P needs a single-domain 1D plan with a fast rule");
        if (max_block_steps(p, 32) < 1 || d.n_local < 32 * 32)
            return fail(FQNM_ERR_UNSUPPORTED, "K2P needs n >= one V = 32 window");
        if (!p->scratch) {
            p->scratch_bytes = state_elems(d) * elem_size(d);
            CUDA_TRY(cudaMalloc(&p->scratch, p->scratch_bytes));
        }
        p->family = 2;
        if (p->k < 1) p->k = 16;
        if (p->k > max_block_steps(p, 32)) p->k = max_block_steps(p, 32);
        p->V = 32;
        p->minb = 2;
        p->persist = 1;
        p->no_sign = !persist_sign;
        if (k) {
            if (k > max_block_steps(p, 32)) return fail(FQNM_ERR_ARG, "k too large for V = 32");
            p->k = k;
        }
        return FQNM_OK;
    }
    if (kernel == 2) { p->persist = 0; p->no_sign = !allow_sign; }
    if (kernel) {
        if (d.boundary == FQNM_HALO && kernel != 2) return fail(FQNM_ERR_UNSUPPORTED, "split domains use K2");
        if (kernel == 3) {
            if (d.n_local % 32 != 0 || !warp_ensemble_has_V((int)(d.n_local / 32)))
                return fail(FQNM_ERR_UNSUPPORTED, "warp ensemble needs n = 32 V, V in {1..32}");
            p->V = (int)(d.n_local / 32);
        } else if (kernel == 4) {
            if (d.n_local > 16384) return fail(FQNM_ERR_UNSUPPORTED, "CTA ensemble needs n <= 16384");
        } else if (kernel == 6) {
            if (d.batch != 1 || d.boundary == FQNM_HALO)
                return fail(FQNM_ERR_UNSUPPORTED, "resident stepper needs one problem, no split");
            int P, base, rem, H;
            const int saveV = p->V, savek = p->k;
            p->V = (V == 4 || V == 8) ? V : 8;
            p->k = p->k > 0 && p->k <= 124 ? p->k : 16;
            int rc6 = resident_geometry(p, p->k, &P, &base, &rem, &H);
            if (rc6 != FQNM_OK) { p->V = saveV; p->k = savek; return fail(rc6, "resident stepper: n not supported"); }
            if ((rc6 = resident_alloc(p)) != FQNM_OK) return rc6;
            if (!p->scratch) {
                p->scratch_bytes = state_elems(d) * elem_size(d);
                CUDA_TRY(cudaMalloc(&p->scratch, p->scratch_bytes));
            }
        } else if (kernel == 1 || kernel == 2) {
            if (!p->scratch && d.boundary != FQNM_HALO) {
                p->scratch_bytes = state_elems(d) * elem_size(d);
                CUDA_TRY(cudaMalloc(&p->scratch, p->scratch_bytes));
            }
            if (kernel == 2 && !p->V) { p->V = 16; p->k = 16; }
            if (kernel == 2 && (p->V < 8 || !blocked_has_V(p->V))) p->V = 16;
            if (kernel == 2 && p->k < 1) p->k = 8;
        } else {
            return fail(FQNM_ERR_ARG, "unknown kernel family %d", kernel);
        }
        p->family = kernel;
    }
    if (V && p->family == 6) {
        V = 0;                           // consumed above
    }
    if (V) {
        if (p->family != 2 || !blocked_rule_has_V(p->rule, V))
            return fail(FQNM_ERR_UNSUPPORTED, "V override needs K2 and V in {8,16,32} ({8,16} for two-point rules)");
        p->V = V;
    }
    if (k && p->family == 6) {
        int P, base, rem, H;
        if (k > 124 || resident_geometry(p, k, &P, &base, &rem, &H) != FQNM_OK || P > p->res_P)
            return fail(FQNM_ERR_ARG, "k = %d not valid for the resident stepper", k);
        p->k = k;
        return FQNM_OK;
    }
    if (k) {
        if (p->family != 2) return fail(FQNM_ERR_UNSUPPORTED, "k override needs K2");
        if (k > max_block_steps(p, p->V)) return fail(FQNM_ERR_ARG, "k too large for V");
        if (d.boundary == FQNM_HALO && k > d.halo) return fail(FQNM_ERR_ARG, "k > halo");
        p->k = k;
    }
    if (p->family == 2 && p->k > max_block_steps(p, p->V)) p->k = max_block_steps(p, p->V);
    return FQNM_OK;
}

extern "C" int64_t fqnm_launch_count(const fqnm_plan_t* p) { return p ? p->launches : 0; }

extern "C" const char* fqnm_last_error(void) { return g_err.c_str(); }

extern "C" const char* fqnm_status_str(int s)
{
    switch (s) {
        case FQNM_OK: return "FQNM_OK";
        case FQNM_ERR_ARG: return "FQNM_ERR_ARG";
        case FQNM_ERR_CFL: return "FQNM_ERR_CFL";
        case FQNM_ERR_RANGE: return "FQNM_ERR_RANGE";
        case FQNM_ERR_CUDA: return "FQNM_ERR_CUDA";
        case FQNM_ERR_UNSUPPORTED: return "FQNM_ERR_UNSUPPORTED";
        case FQNM_ERR_NOMEM: return "FQNM_ERR_NOMEM";
        default: return "FQNM_ERR_UNKNOWN";
    }
}

extern "C" int fqnm_abi_version(void) { return FQNM_ABI_VERSION; }
