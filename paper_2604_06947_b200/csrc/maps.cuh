// Device evaluation of the integer transfer maps phi+(q), phi-(q)
// (Eq. flux_table) for the rule the planner selected.
//
// Every variant returns exactly round((c2 q^2 + c1 q)/den) of the plan's exact
// rational map (reading D2); the fast variants are closed forms whose validity
// range the planner proves before selecting them.
#pragma once

#include <cstdint>
#include "fqnm_internal.h"

// EO pipe-balance variant (tools/tune_variants.sh, profiles/r01_tune_eo_variants*.jsonl):
// 3 = conversion by I2FP and phi- by LOP3 (12.2 instr/cell, measured fastest on B200),
// 2 = conversion by IMAD + FADD, 1 = conversion by LOP3 + FADD, 0/4 = phi- by IMAD.
#ifndef FQNM_EO_VARIANT
#define FQNM_EO_VARIANT 3
#endif

namespace fqnm {

// round(num/den) for den > 0 in int64 (headroom validated by the planner)
__device__ __forceinline__ int64_t round_div_i64(int64_t num, int64_t den, int rounding)
{
    if (rounding == 1) {                         // FLOOR
        int64_t qt = num / den;
        if ((num % den != 0) && (num < 0)) qt -= 1;
        return qt;
    }
    int64_t a = num < 0 ? -num : num;
    int64_t r;
    if (rounding == 0) {                         // half away from zero
        r = (2 * a + den) / (2 * den);
    } else {                                     // half to even
        int64_t fl = a / den, rem = a - fl * den;
        if (2 * rem > den) r = fl + 1;
        else if (2 * rem < den) r = fl;
        else r = (fl & 1) ? fl + 1 : fl;
    }
    return num < 0 ? -r : r;
}

// RHA(num / den) in float64 for |num| < 2^44 (planner), instead of a 64-bit division:
//   X = bits(1.5 2^52) + num is the double 1.5 2^52 + num exactly (|num| < 2^51);
//   t = fma(X, d, -1.5 2^52 d) = fl(num d), d = (1/den)(1 + 2^-46) with its last two significand
//       bits cleared so that 1.5 2^52 d is exact; the relative bias b of t, 2^-47 < b < 2^-45, moves
//       v = num/den away from zero: an exact tie rounds away from zero (RHA), and any other v
//       is >= 1/(2 den) from a half-integer while |v| b < 2^-45 |num| / den < 1/(2 den);
//   result = low word of bits(t + 1.5 2^52) (two's complement of rint(t), |result| < 2^31).
__device__ __forceinline__ int32_t round_div_dp(int64_t num, double dinv, double dc)
{
    const double X = __longlong_as_double(num + 0x4338000000000000ll);
    const double t = __fma_rn(X, dinv, dc);
    return __double2loint(__dadd_rn(t, 6755399441055744.0));
}

__device__ __forceinline__ int32_t generic_phi(int32_t q, int64_t c2, int64_t c1, int64_t den,
                                               int32_t supp, int rounding)
{
    if (supp == SUPP_NONE) return 0;
    if (supp == SUPP_POS && q <= 0) return 0;
    if (supp == SUPP_NEG && q >= 0) return 0;
    int64_t qq = q;
    int64_t num = c2 * qq * qq + c1 * qq;
    return (int32_t)round_div_i64(num, den, rounding);
}

// the same with the float64 division where the planner allows it (which: 0 phi+, 1 phi-)
__device__ __forceinline__ int32_t generic_phi_sel(int32_t q, int64_t c2, int64_t c1, int64_t den,
                                                   int32_t supp, const DevRule& r, int which)
{
    if (!r.dv_ok[which]) return generic_phi(q, c2, c1, den, supp, r.rounding);
    if (supp == SUPP_NONE) return 0;
    if (supp == SUPP_POS && q <= 0) return 0;
    if (supp == SUPP_NEG && q >= 0) return 0;
    const int64_t qq = q;
    return round_div_dp(c2 * qq * qq + c1 * qq, r.dv_inv[which], r.dv_c[which]);
}

__device__ __forceinline__ int32_t imad_hi(int32_t a, int32_t b, int32_t c)
{
    // ((int64) a * b >> 32) + c on the FMA pipe; with b = 1: c + (a >> 31)
    int32_t d;
    asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// EO Burgers magnitude g(q) = floor((2P q^2 + Q) / (2Q)) = RHA(kappa q^2),
// for |q| < 2^22 and kappa q^2 <= 2^20 (proved at plan time):
// 1. qf = float(q) exactly via the 1.5*2^23 magic (IADD + FADD);
//    est = rint(fl(qf*qf) * cf) with cf <= kappa (1 - 2^-21) rounded down, done
//    by one FFMA into the 1.5*2^23 magic: the relative underestimate keeps
//    est in {g - 1, g} (never above g, at most one below).
// 2. u = 2Q - 1 - r with r = 2P q^2 + Q - 2Q est, evaluated modulo 2^32 (exact:
//    0 <= r < 4Q < 2^31); est is one short exactly when r >= 2Q, i.e. u < 0.
//    Constants: eo_c1 = Q - 1 - 2Q*0x4B400000 (mod 2^32), eo_ntwoP = -2P, eo_twoQ = 2Q.
__device__ __forceinline__ uint32_t lop3_6c(uint32_t a, uint32_t b, uint32_t c)
{
    // d = c ? (a ^ b) : b   (LUT 0x6C with a = 0xF0, b = 0xCC, c = 0xAA)
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x6C;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ int32_t imad(int32_t a, int32_t b, int32_t c)
{
    // a*b + c on the FMA pipe (ptxas keeps an IMAD when b is not a known constant)
    int32_t d;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Per cell, variant 3: I2FP, FMUL, FFMA, 4 IMAD (q^2, 2 x remainder,
// -K), LEA.HI, SHF, LOP3 and the step's 2 x IADD3 -> 12 SASS instructions.
__device__ __forceinline__ void eo_gm(int32_t q, int32_t& g, int32_t& m, const DevRule& r)
{
    // 0x4B400000 + q for |q| < 2^22 as one LOP3: bits 0..22 of q with bit 22
    // flipped, exponent/sign bits of 1.5*2^23 above
#if FQNM_EO_VARIANT >= 3
    const float qf = __int2float_rn(q);                                  // exact, |q| < 2^24
#elif FQNM_EO_VARIANT == 2
    const uint32_t x = (uint32_t)imad(q, r.one, 0x4B400000);
    const float qf = __int_as_float((int32_t)x) - 12582912.0f;          // exact
#else
    const uint32_t x = lop3_6c((uint32_t)q, 0x4B400000u, 0x007FFFFFu);
    const float qf = __int_as_float((int32_t)x) - 12582912.0f;          // exact
#endif
    const float s = __fmul_rn(qf, qf);
    const float t = __fmaf_rn(s, r.eo_cf, 12582912.0f);                 // 0x4B400000 + est
    const int32_t bits = __float_as_int(t);
    const int32_t q2 = imad(q, q, 0);                                    // q^2 mod 2^32
    int32_t u = imad(q2, r.eo_ntwoP, r.eo_c1);
    u = imad(bits, r.eo_twoQ, u);                                        // 2Q - 1 - r
    const int32_t gb = bits + (int32_t)((uint32_t)u >> 31);              // LEA.HI
    g = imad(gb, r.one, (int32_t)0xB4C00000);                            // - 0x4B400000
#if FQNM_EO_VARIANT == 0 || FQNM_EO_VARIANT == 4
    m = imad(g, (int32_t)((uint32_t)q >> 31), 0);                        // phi-(q) = [q<0] g
#else
    m = g & (q >> 31);
#endif
}

// EO magnitude for P = 1 (kappa = 1/Q; every EO plan of BJ has P = 1), two
// instructions shorter than eo_gm:
// 1. est is estimated as in eo_gm but with the magic 1.5*2^23 + 1, so
//    bits = 0x4B400000 + 1 + est, est in {g - 1, g} (the tie rule of the FFMA
//    does not matter: est is floor or ceil of a strict underestimate).
// 2. est = g - 1 exactly when v = P q^2 - Q est - ceil(Q/2) >= 0 (integers:
//    2Pq^2 + Q >= 2Q(est + 1)); |v| < 2Q, so v is exact modulo 2^32:
//    v = q*q + (-Q)*bits + c6,  c6 = Q*(0x4B400000 + 1) - ceil(Q/2).
// 3. gb = bits + (v >> 31) = 0x4B400000 + g  (LEA.HI.SX32), and since g < 2^22
//    the bias sits above bit 21: g = gb & 0x3FFFFF, phi-(q) = gb & 0x3FFFFF & (q >> 31)
//    in one LOP3.  BIASED returns gb itself as g: the step only uses differences of
//    interface transfers, so a constant bias in g (never in m) cancels.
// CONV selects the exact int -> float conversion: I2FP (ALU pipe) or IMAD + FADD
// (FMA pipe), so cells can alternate to balance the two pipes.
template <int CONV, bool BIASED>
__device__ __forceinline__ void eo_gm_p1(int32_t q, int32_t& g, int32_t& m, const DevRule& r)
{
    float qf;
    if (CONV == 0) qf = __int2float_rn(q);                               // exact, |q| < 2^24
    else qf = __int_as_float(imad(q, r.one, 0x4B400000)) - 12582912.0f;   // exact, |q| < 2^22
    const float s = __fmul_rn(qf, qf);
    const float t = __fmaf_rn(s, r.eo_cf, 12582913.0f);                 // 0x4B400001 + est
    const int32_t bits = __float_as_int(t);
    const int32_t v = imad(bits, r.eo_nQ, imad(q, q, r.eo_c6));          // q*q off the float chain
    const int32_t gb = bits + (v >> 31);                                 // 0x4B400000 + g
#if FQNM_EO_P1_SIGN
    const int32_t sg = __mulhi(q, r.one);                                // q >> 31 as IMAD.HI (FMA pipe)
#else
    const int32_t sg = q >> 31;
#endif
    m = gb & 0x3FFFFF & sg;                                              // [q<0] g
    g = BIASED ? gb : (gb & 0x3FFFFF);
}

// EO magnitude alone, for sign-uniform windows (DESIGN.md §K2 "sign-uniform windows"):
// where every cell of a window has q >= 0, phi-(q) = 0 and phi+(q) = g(q) (the EO split's
// supports, P:62-68 with f- = min(u,0)^2/2), so the step needs g only; q <= 0 likewise
// needs g = phi- only.  Returns g with the constant bias of eo_gm_p1 for P = 1 (the
// step uses differences of g only).  P = 1: I2FP (or IMAD + FADD, CONV = 1), FMUL,
// FFMA, 2 IMAD, LEA.HI = 6 instructions, against eo_gm_p1's 8.
#ifndef FQNM_EO_SIGN_LEA
#define FQNM_EO_SIGN_LEA 0     // bits + (v >> 31): 0 LEA.HI (ALU pipe), 1 IMAD.HI (FMA pipe), 2 alternate
#endif
#ifndef FQNM_EO_SIGN_CONV
#define FQNM_EO_SIGN_CONV 0    // 0: I2FP for every cell, 1: IMAD + FADD, 2: alternate by cell
#endif
// EO magnitude map in float64, 4 instructions with the update (IMAD.WIDE, DFMA, DADD + the
// step's IADD3) against 7 for the float32-estimate + integer-remainder form.
//   X  = q*q + bits(2^52)  is the double 2^52 + q^2 exactly (ulp(2^52) = 1, q^2 < 2^44: one IMAD.WIDE makes
//        the product and the int64 -> double conversion);
//   t1 = fma(X, dinv, -2^52 dinv) = fl(q^2 dinv): the FMA forms X dinv - 2^52 dinv = q^2 dinv
//        exactly and rounds once, so t1 = v (1 + b), v = P q^2 / Q, 2^-47 < b < 2^-45
//        (dinv = (P/Q)(1 + 2^-46) up to 2^-52, the rounding 2^-53);
//   g  = low word of bits(t1 + 1.5 2^52) = rint(t1).
// rint(t1) = RHA(v) = floor(v + 1/2): a tie v = k + 1/2 is pushed up by v b >= 16 ulp(v), so it
// rounds to k + 1; any other v is at least 1/(2Q) from a half-integer and v b < 2^-45 v <
// 1/(2Q) because v Q = P q^2 < 2^44 (eo_dp_ok, checked by the planner on the admissible
// range), so t1 stays on v's side of every boundary and is never a half-integer itself.
#ifndef FQNM_EO_DP
#define FQNM_EO_DP 1           // sign-uniform EO step (P = 1): 1 = the float64 form (cfg4 4.18 -> 4.5 TCUPS)
#endif
__device__ __forceinline__ int32_t eo_g_dp(int32_t q, const DevRule& r)
{
    const long long X = (long long)q * (long long)q + r.eo_xoff;
    const double t1 = __fma_rn(__longlong_as_double(X), r.eo_dinv, r.eo_dc1);
    return __double2loint(__dadd_rn(t1, 6755399441055744.0));
}

template <int RULE, bool ALT>
__device__ __forceinline__ int32_t eo_g_biased(int32_t q, const DevRule& r);
// the EO magnitude of the sign-uniform steps: the float64 form for P = 1 (P q^2 < 2^44 holds
// on the whole fast-path domain |q| < 2^22, eo_dp_ok; g unbiased) unless F32 asks for the
// float32 + integer-remainder form (g biased for P = 1; a step uses one form throughout)
template <int RULE, bool ALT, bool F32>
__device__ __forceinline__ int32_t eo_g_sel(int32_t q, const DevRule& r)
{
    if (FQNM_EO_DP && !F32 && RULE == R_EO_P1) return eo_g_dp(q, r);
    return eo_g_biased<RULE, ALT>(q, r);
}

template <int RULE, bool ALT>
__device__ __forceinline__ int32_t eo_g_biased(int32_t q, const DevRule& r)
{
    if (RULE == R_EO_P1) {
        constexpr bool fma_conv = FQNM_EO_SIGN_CONV == 1 || (FQNM_EO_SIGN_CONV == 2 && ALT);
        float qf;
        if (!fma_conv) qf = __int2float_rn(q);                               // exact, |q| < 2^24
        else qf = __int_as_float(imad(q, r.one, 0x4B400000)) - 12582912.0f;  // exact, |q| < 2^22
        const float s = __fmul_rn(qf, qf);
        const float t = __fmaf_rn(s, r.eo_cf, 12582913.0f);                 // 0x4B400001 + est
        const int32_t bits = __float_as_int(t);
        // v = q*q + (-Q) bits + c6 (mod 2^32) with q*q + c6 first: that IMAD does not wait
        // for the float chain, so the chain's tail is one IMAD + LEA (micro: 0.90 vs 0.81 issue)
        const int32_t v = imad(bits, r.eo_nQ, imad(q, q, r.eo_c6));
        constexpr bool hi_fma = FQNM_EO_SIGN_LEA == 1 || (FQNM_EO_SIGN_LEA == 2 && ALT);
        if (hi_fma) return imad_hi(v, r.one, bits);                          // FMA pipe
        return bits + (v >> 31);                                             // 0x4B400000 + g (LEA.HI)
    } else {
        int32_t g, m;
        eo_gm(q, g, m, r);
        return g;
    }
}

// LINEAR |kappa| = P/Q <= 1: phi(q) = sign(kappa q) floor((2P|q| + Q)/(2Q)), for
// |q| < 2^24 and |kappa q| <= 2^20 (planner), with the EO scheme: est = rint(|q_f| cf)
// (one FFMA, cf <= |kappa|(1 - 2^-21)) is g or g - 1, corrected by the sign of
// u = 2Q - 1 - (2P|q| + Q - 2Q est) computed modulo 2^32.
__device__ __forceinline__ int32_t lin_phi(int32_t q, const DevRule& r)
{
    const float af = fabsf(__int2float_rn(q));                            // exact
    const float t = __fmaf_rn(af, r.eo_cf, 12582912.0f);                 // 0x4B400000 + est
    const int32_t bits = __float_as_int(t);
    const int32_t a = q < 0 ? -q : q;
    int32_t u = imad(a, r.eo_ntwoP, r.eo_c1);
    u = imad(bits, r.eo_twoQ, u);
    const int32_t g = imad(bits + (int32_t)((uint32_t)u >> 31), r.one, (int32_t)0xB4C00000);
    const int32_t sgn = q >> 31;                                          // -1 for q < 0
    return (g ^ sgn) - sgn;                                               // sign(q) g
}

// (g, m) with g = phi+(q) + phi-(q) and m = phi-(q); phi+(q) = g - m.
// The step uses F_{j+1/2} = phi+(q_j) + phi-(q_{j+1}) = g_j - m_j + m_{j+1} (one IADD3).
#ifndef FQNM_EO_P1_SIGN
#define FQNM_EO_P1_SIGN 0      // sign mask q >> 31: 0 SHF (ALU pipe), 1 IMAD.HI (FMA pipe)
#endif
#ifndef FQNM_EO_P1_CONV
#define FQNM_EO_P1_CONV 2      // 0: I2FP, 1: IMAD + FADD, 2: alternate by cell parity (fastest, profiles/r01_tune_eo_p1.jsonl)
#endif

// BIASED: g may carry a constant bias (see eo_gm_p1); only the stepping kernels,
// which use differences of g, ask for it
template <int RULE, bool ALT = false, bool BIASED = false>
__device__ __forceinline__ void phi_gm(int32_t q, int32_t& g, int32_t& m, const DevRule& r)
{
    if (RULE == R_LIN_HALF) {
        // RHA(q/2) = q - trunc(q/2) for every signed q (C division truncates)
        g = q - q / 2;
        m = 0;
    } else if (RULE == R_EO_FAST) {
        eo_gm(q, g, m, r);               // phi-(q) = g for q < 0, phi+(q) = g for q > 0, g(0) = 0
    } else if (RULE == R_EO_P1) {
        eo_gm_p1<(FQNM_EO_P1_CONV == 1 || (FQNM_EO_P1_CONV == 2 && ALT)) ? 1 : 0, BIASED>(q, g, m, r);
    } else if (RULE == R_LIN_FAST) {
        // a > 0: phi+ = RHA(kappa q) = v, phi- = 0;  a < 0: phi+ = 0, phi- = RHA(kappa q) = -v
        const int32_t v = lin_phi(q, r);
        if (r.lin_minus) { g = -v; m = -v; }
        else { g = v; m = 0; }
    } else {
        const int32_t p = generic_phi_sel(q, r.c2p, r.c1p, r.denp, r.suppp, r, 0);
        m = generic_phi_sel(q, r.c2m, r.c1m, r.denm, r.suppm, r, 1);
        g = p + m;
    }
}

template <int RULE>
__device__ __forceinline__ void phi_pm(int32_t q, int32_t& p, int32_t& m, const DevRule& r)
{
    int32_t g;
    phi_gm<RULE>(q, g, m, r);
    p = g - m;
}

// Quantised two-point transfer rule, rounded once (Thm transfer-operator
// equivalence; include/fqnm.h FQNM_BURGERS_GODUNOV/EO2/LF2):
// Phi(qL, qR) = round(num / den) with num from the plan's integer coefficients,
// evaluated exactly in int64 (headroom validated by the planner).
__device__ __forceinline__ int32_t tp_phi(int32_t qL, int32_t qR, const DevRule& r)
{
    const int64_t L = qL, R = qR;
    int64_t num;
    if (r.tp_kind == 7) {
        num = r.tp_c2 * (L * L + R * R) + r.tp_c1 * (L - R);
    } else {
        const int64_t a = L > 0 ? L : 0, b = R < 0 ? R : 0;
        const int64_t A = a * a, B = b * b;
        num = r.tp_c2 * (r.tp_kind == 5 ? (A > B ? A : B) : A + B);
    }
    if (r.dv_ok[2]) return round_div_dp(num, r.dv_inv[2], r.dv_c[2]);
    return (int32_t)round_div_i64(num, r.tp_den, r.rounding);
}

// Godunov for Burgers on the EO fast path's domain (rule R_TP_FAST):
// Phi = RHA(kappa max(max(qL,0)^2, min(qR,0)^2)) = g(x), x = max(max(qL,0), -min(qR,0)),
// with the EO magnitude g in closed form (exact for |q| < 2^22, kappa q^2 <= 2^20,
// proved by the planner); tp_fast = 1: P = 1 form, 2: general P
__device__ __forceinline__ int32_t tp_godunov_fast(int32_t qL, int32_t qR, const DevRule& r)
{
    const int32_t a = qL > 0 ? qL : 0, b = qR < 0 ? -qR : 0;
    const int32_t x = a > b ? a : b;
    int32_t g, m;
    if (r.tp_fast == 1) eo_gm_p1<0, false>(x, g, m, r);
    else eo_gm(x, g, m, r);
    return g;
}

template <int RULE>
__device__ __forceinline__ int32_t tp_eval(int32_t qL, int32_t qR, const DevRule& r)
{
    if (RULE == R_TP_FAST) return tp_godunov_fast(qL, qR, r);
    return tp_phi(qL, qR, r);
}

// Interface transfer T = Phi(qL, qR) of any scalar rule: split rules
// phi+(qL) + phi-(qR), two-point rules tp_phi.
template <int RULE>
__device__ __forceinline__ int32_t transfer_lr(int32_t qL, int32_t qR, const DevRule& r)
{
    if (RULE == R_TWOPOINT || RULE == R_TP_FAST) return tp_eval<RULE>(qL, qR, r);
    int32_t pL, mL, pR, mR;
    phi_pm<RULE>(qL, pL, mL, r);
    phi_pm<RULE>(qR, pR, mR, r);
    return pL + mR;
}

// 2D/3D range guard: a stored cell outside the plan's admissible range [lo, hi] (where
// the fast closed-form maps are proven exact) flags the call (fqnm_api.cu md_guard_*)
__device__ __forceinline__ void md_note(int* guard, int32_t v, int32_t lo, int32_t hi)
{
    if (guard && (v < lo || v > hi)) atomicOr(guard, 1);
}
// the same guard without a branch per cell: acc = max over cells of (unsigned)(v - lo); the
// cell is outside [lo, hi] exactly when that exceeds hi - lo (v < lo wraps to a huge value).
// One add + one max per cell, one test per thread at the end of its chunk (md_flush).
__device__ __forceinline__ void md_acc(unsigned& acc, int32_t v, int32_t lo)
{
    const unsigned d = (unsigned)v - (unsigned)lo;
    acc = d > acc ? d : acc;
}
__device__ __forceinline__ void md_flush(int* guard, unsigned acc, int32_t lo, int32_t hi)
{
    if (guard && acc > (unsigned)hi - (unsigned)lo) atomicOr(guard, 1);
}

}  // namespace fqnm
