// Device evaluation of the integer transfer maps phi+(q), phi-(q)
// (Eq. flux_table) for the rule the planner selected.
//
// Every variant returns exactly round((c2 q^2 + c1 q)/den) of the plan's exact
// rational map (reading D2); the fast variants are closed forms whose validity
// range the planner proves before selecting them.
#pragma once

#include <cstdint>
#include "fqnm_internal.h"

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

// EO Burgers magnitude g(a) = floor((2P a^2 + Q) / (2Q)), a = |q| < 2^23.
// 1. est = nearest integer to fl(fl(a*a) * fl(P/Q)) via the 1.5*2^23 magic add
//    (one rounding inside the FMA); |est - g| <= 1 while kappa a^2 < 2^22.
// 2. rem = 2P a^2 + Q - 2Q est is computed modulo 2^32 and is exact because
//    -2Q <= rem < 4Q < 2^31 (Q < 2^29); one correction step in each direction.
__device__ __forceinline__ int32_t eo_g(int32_t q, const DevRule& r)
{
    uint32_t a = (uint32_t)(q < 0 ? -q : q);
    float af = __int_as_float((int32_t)(0x4B000000u | a)) - 8388608.0f;   // exact, a < 2^23
    float s = __fmul_rn(af, af);
    float t = __fmaf_rn(s, r.eo_cf, 12582912.0f);
    int32_t est = __float_as_int(t) - 0x4B400000;
    uint32_t a2 = a * a;
    int32_t rem = (int32_t)(a2 * (uint32_t)r.eo_twoP + (uint32_t)r.eo_Q
                            - (uint32_t)est * (uint32_t)r.eo_twoQ);
    est += (rem >> 31);                                    // rem < 0   -> est - 1
    est += (int32_t)((uint32_t)(r.eo_twoQ - 1 - rem) >> 31);   // rem >= 2Q -> est + 1
    return est;
}

template <int RULE>
__device__ __forceinline__ void phi_pm(int32_t q, int32_t& p, int32_t& m, const DevRule& r)
{
    if (RULE == R_LIN_HALF) {
        // RHA(q/2) = q - trunc(q/2) for every signed q (C division truncates)
        p = q - q / 2;
        m = 0;
    } else if (RULE == R_EO_FAST) {
        int32_t g = eo_g(q, r);
        int32_t neg = q >> 31;          // -1 when q < 0
        m = g & neg;                     // phi-(q) = g for q < 0
        p = g - m;                       // phi+(q) = g for q > 0 (g(0) = 0)
    } else {
        p = generic_phi(q, r.c2p, r.c1p, r.denp, r.suppp, r.rounding);
        m = generic_phi(q, r.c2m, r.c1m, r.denm, r.suppm, r.rounding);
    }
}

}  // namespace fqnm
