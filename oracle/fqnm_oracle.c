/*
 * FQNM CPU oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of the FQNM update of
 * arXiv 2604.06947 (PAPER.md, cited as P:line).  Only tests/, the smoke check
 * in __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no source with the CUDA path
 * (paper_2604_06947_b200/csrc, include/), and nothing here is called by the
 * product path.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *        (no FMA contraction: the Roe path pins every binary64 operation).
 *
 * Contents
 *   1. rounding of an exact rational            (Eq. flux_table, readings A1/D1/D2)
 *   2. the integer transfer maps phi+/-         (Eq. flux_table)
 *   3. interface count flux + conservative update, flux-difference form
 *                                               (Eqs. 7-8) and the
 *      four-term form                           (Eq. update_rule)
 *   4. reconstruction u = delta q               (Eq. reconstruction_operator)
 *   5. quantised two-point Roe transfer for the Euler system
 *                                               (Thm transfer-operator equivalence
 *      Eq. applied componentwise; Roe flux structure P:567,
 *      operation order pinned by SURVEY §8(c)-C2 / DESIGN.md reading R-ROE)
 *
 * A transfer map is a piecewise polynomial of degree <= 2 with exact rational
 * coefficients, i.e. phi(q) = [q in support] * round( (c2 q^2 + c1 q) / D ),
 * which is f(delta q) * (dt/dx) / delta written over a common denominator D
 * (the coefficients are produced from the paper's formula by exact Fraction
 * arithmetic in oracle/rules.py).  Every intermediate is a 128-bit integer.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef __int128 i128;

/* rounding rules (reading A1): RHA is the default; FLOOR is the literal
 * mean-field closure n = floor(Np) of Eq. mean_field_closure;
 * HALF_EVEN is the other common tie rule.  Same codes as include/fqnm.h. */
enum { OR_RHA = 0, OR_FLOOR = 1, OR_HALF_EVEN = 2 };

/* support of a map: all q, q > 0 only, q < 0 only */
enum { OR_SUPP_ALL = 0, OR_SUPP_POS = 1, OR_SUPP_NEG = 2 };

typedef struct {
    int64_t c2, c1, den;   /* phi(q) = round((c2 q^2 + c1 q)/den), den > 0 */
    int32_t support;
    int32_t rounding;
} or_map;

/* ---- 1. rounding of the exact rational num/den (den > 0) --------------- */
static i128 floor_div(i128 num, i128 den)
{
    i128 q = num / den;            /* C truncates toward zero */
    if ((num % den != 0) && (num < 0)) q -= 1;
    return q;
}

int64_t or_round_rational(int64_t num_hi, uint64_t num_lo, int64_t den, int rounding)
{
    i128 num = ((i128)num_hi << 64) | (i128)num_lo;
    i128 d = den;
    if (rounding == OR_FLOOR) return (int64_t)floor_div(num, d);
    i128 a = num < 0 ? -num : num;
    if (rounding == OR_RHA) {
        /* RHA(x) = sign(x) floor(|x| + 1/2) */
        i128 r = (2 * a + d) / (2 * d);
        return (int64_t)(num < 0 ? -r : r);
    }
    /* half-to-even on |x|, then restore sign */
    i128 fl = a / d, rem = a - fl * d;
    i128 r;
    if (2 * rem > d) r = fl + 1;
    else if (2 * rem < d) r = fl;
    else r = (fl % 2 == 0) ? fl : fl + 1;
    return (int64_t)(num < 0 ? -r : r);
}

/* ---- 2. transfer map phi(q) (Eq. flux_table) ---------------------------- */
int64_t or_phi(const or_map* m, int64_t q)
{
    if (m->support == OR_SUPP_POS && !(q > 0)) return 0;
    if (m->support == OR_SUPP_NEG && !(q < 0)) return 0;
    i128 num = (i128)m->c2 * (i128)q * (i128)q + (i128)m->c1 * (i128)q;
    i128 d = m->den;
    if (m->rounding == OR_FLOOR) return (int64_t)floor_div(num, d);
    i128 a = num < 0 ? -num : num;
    if (m->rounding == OR_RHA) {
        i128 r = (2 * a + d) / (2 * d);
        return (int64_t)(num < 0 ? -r : r);
    }
    i128 fl = a / d, rem = a - fl * d, r;
    if (2 * rem > d) r = fl + 1;
    else if (2 * rem < d) r = fl;
    else r = (fl % 2 == 0) ? fl : fl + 1;
    return (int64_t)(num < 0 ? -r : r);
}

void or_phi_array(const or_map* m, const int64_t* q, int64_t* out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) out[i] = or_phi(m, q[i]);
}

/* ---- 3. one explicit step ------------------------------------------------ */
enum { OR_PERIODIC = 0, OR_TRANSMISSIVE = 1 };

/* interface count flux F_{i+1/2} = phi+(q_i) + phi-(q_{i+1}) for
 * i = -1 .. N-1.  Periodic: q_{-1} = q_{N-1}, q_N = q_0.  Transmissive
 * (reading A12): ghost cells copy the edge cell, q_{-1} = q_0, q_N = q_{N-1}. */
static int64_t flux_at(const or_map* pp, const or_map* pm, int boundary,
                       int64_t N, const int64_t* q, int64_t i)
{
    int64_t iL = i, iR = i + 1;
    if (boundary == OR_PERIODIC) {
        if (iL < 0) iL += N;
        if (iR >= N) iR -= N;
    } else {
        if (iL < 0) iL = 0;
        if (iR >= N) iR = N - 1;
    }
    return or_phi(pp, q[iL]) + or_phi(pm, q[iR]);
}

/* q^{n+1}_i = q^n_i - (F_{i+1/2} - F_{i-1/2})  (Eq. update_rule_conservative_form,
 * P:86-89).  All fluxes are evaluated on q^n (explicit update, reading D6). */
void or_step_scalar(const or_map* pp, const or_map* pm, int boundary, int64_t N,
                    const int64_t* q, int64_t* out)
{
    #pragma omp parallel for schedule(static) if (N >= 32768)
    for (int64_t i = 0; i < N; ++i) {
        int64_t Fr = flux_at(pp, pm, boundary, N, q, i);
        int64_t Fl = flux_at(pp, pm, boundary, N, q, i - 1);
        out[i] = q[i] - (Fr - Fl);
    }
}

/* The four-term form of Eq. update_rule, periodic only:
 * q_i - (phi+(q_i) + phi-(q_{i+1}) - phi+(q_{i-1}) - phi-(q_i)). */
void or_step_scalar_fourterm(const or_map* pp, const or_map* pm, int64_t N,
                             const int64_t* q, int64_t* out)
{
    for (int64_t i = 0; i < N; ++i) {
        int64_t im = (i == 0) ? N - 1 : i - 1;
        int64_t ip = (i == N - 1) ? 0 : i + 1;
        out[i] = q[i] - (or_phi(pp, q[i]) + or_phi(pm, q[ip])
                         - or_phi(pp, q[im]) - or_phi(pm, q[i]));
    }
}

/* nsteps explicit steps, double buffered.  q is updated in place. */
static void run_one(const or_map* pp, const or_map* pm, int boundary, int64_t N,
                    int64_t* q, int64_t nsteps)
{
    int64_t* a = q;
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    for (int64_t s = 0; s < nsteps; ++s) {
        or_step_scalar(pp, pm, boundary, N, a, b);
        int64_t* t = a; a = b; b = t;
    }
    if (a != q) { memcpy(q, a, sizeof(int64_t) * (size_t)N); b = a; }
    free(b);
}

static void set_threads(int nthreads)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

/* nthreads <= 0 leaves the OpenMP default. */
void or_run_scalar(const or_map* pp, const or_map* pm, int boundary, int64_t N,
                   int64_t* q, int64_t nsteps, int nthreads)
{
    set_threads(nthreads);
    run_one(pp, pm, boundary, N, q, nsteps);
}

/* Batched independent problems [B][N] (ensemble mode), one problem per thread. */
void or_run_scalar_batch(const or_map* pp, const or_map* pm, int boundary, int64_t B,
                         int64_t N, int64_t* q, int64_t nsteps, int nthreads)
{
    set_threads(nthreads);
    #pragma omp parallel for schedule(dynamic) if (B > 1)
    for (int64_t b = 0; b < B; ++b)
        run_one(pp, pm, boundary, N, q + b * N, nsteps);
}

/* ---- 3a. quantised two-point transfer rules ------------------------------- */
/* Thm transfer-operator equivalence: Phi(qL, qR) =
 * round(F(delta qL, delta qR) dt/dx / delta) for a classical two-point flux F,
 * rounded once (Eq. transfer_operator_equivalence_definition).
 * Kinds (include/fqnm.h codes): 5 Godunov, 6 EO rounded once, 7 LF rounded once,
 * with integer coefficients from oracle/rules.py (two_point_coefficients):
 *   Godunov: c2 max(max(qL,0)^2, min(qR,0)^2) / den
 *   EO2:     c2 (max(qL,0)^2 + min(qR,0)^2) / den
 *   LF2:     (c2 (qL^2 + qR^2) + c1 (qL - qR)) / den
 * A split rule (kind 0) is the paper's F = phi+(qL) + phi-(qR). */
typedef struct {
    int32_t kind;          /* 0 split, 5/6/7 two-point */
    int32_t rounding;
    int64_t c2, c1, den;   /* two-point coefficients */
    or_map pp, pm;         /* split maps */
} or_transfer;

static int64_t or_round_i128(i128 num, i128 d, int rounding)
{
    if (rounding == OR_FLOOR) return (int64_t)floor_div(num, d);
    i128 a = num < 0 ? -num : num;
    if (rounding == OR_RHA) {
        i128 r = (2 * a + d) / (2 * d);
        return (int64_t)(num < 0 ? -r : r);
    }
    i128 fl = a / d, rem = a - fl * d, r;
    if (2 * rem > d) r = fl + 1;
    else if (2 * rem < d) r = fl;
    else r = (fl % 2 == 0) ? fl : fl + 1;
    return (int64_t)(num < 0 ? -r : r);
}

int64_t or_transfer_eval(const or_transfer* t, int64_t qL, int64_t qR)
{
    if (t->kind == 0) return or_phi(&t->pp, qL) + or_phi(&t->pm, qR);
    i128 L = qL, R = qR, num;
    i128 a = L > 0 ? L : 0, b = R < 0 ? R : 0;
    if (t->kind == 5) num = (i128)t->c2 * (a * a > b * b ? a * a : b * b);
    else if (t->kind == 6) num = (i128)t->c2 * (a * a + b * b);
    else num = (i128)t->c2 * (L * L + R * R) + (i128)t->c1 * (L - R);
    return or_round_i128(num, t->den, t->rounding);
}

void or_transfer_array(const or_transfer* t, const int64_t* qL, const int64_t* qR, int64_t* out,
                       int64_t n)
{
    for (int64_t i = 0; i < n; ++i) out[i] = or_transfer_eval(t, qL[i], qR[i]);
}

/* interface transfer T_{i+1/2} = Phi(q_i, q_{i+1}), i = -1 .. N-1, ghosts as flux_at */
static int64_t transfer_at(const or_transfer* t, int boundary, int64_t N, const int64_t* q,
                           int64_t i)
{
    int64_t iL = i, iR = i + 1;
    if (boundary == OR_PERIODIC) {
        if (iL < 0) iL += N;
        if (iR >= N) iR -= N;
    } else {
        if (iL < 0) iL = 0;
        if (iR >= N) iR = N - 1;
    }
    return or_transfer_eval(t, q[iL], q[iR]);
}

/* q^{n+1}_i = q^n_i - (T_{i+1/2} - T_{i-1/2})  (P:86-89 with F replaced by Phi) */
void or_step_transfer(const or_transfer* t, int boundary, int64_t N, const int64_t* q,
                      int64_t* out)
{
    #pragma omp parallel for schedule(static) if (N >= 32768)
    for (int64_t i = 0; i < N; ++i)
        out[i] = q[i] - (transfer_at(t, boundary, N, q, i) - transfer_at(t, boundary, N, q, i - 1));
}

void or_run_transfer(const or_transfer* t, int boundary, int64_t N, int64_t* q, int64_t nsteps,
                     int nthreads)
{
    set_threads(nthreads);
    int64_t* a = q;
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    for (int64_t s = 0; s < nsteps; ++s) {
        or_step_transfer(t, boundary, N, a, b);
        int64_t* x = a; a = b; b = x;
    }
    if (a != q) { memcpy(q, a, sizeof(int64_t) * (size_t)N); b = a; }
    free(b);
}

/* ---- 3b. Cartesian extension by directional composition ------------------ */
/* Thm formal Cartesian dimensional extension, d = 2, unsplit:
 *   q'_{i,j} = q_{i,j} - (F^x_{i+1/2,j} - F^x_{i-1/2,j}) - (F^y_{i,j+1/2} - F^y_{i,j-1/2}),
 *   F^x_{i+1/2,j} = phi+_x(q_{i,j}) + phi-_x(q_{i+1,j}),
 *   F^y_{i,j+1/2} = phi+_y(q_{i,j}) + phi-_y(q_{i,j+1}),
 * all on q^n.  Layout q[j * nx + i] (x fastest).  Boundaries per direction as
 * in 1D (periodic wrap or transmissive ghost copies). */
static int64_t at2(const int64_t* q, int boundary, int64_t nx, int64_t ny, int64_t i, int64_t j)
{
    if (boundary == OR_PERIODIC) {
        i = (i % nx + nx) % nx;
        j = (j % ny + ny) % ny;
    } else {
        i = i < 0 ? 0 : (i >= nx ? nx - 1 : i);
        j = j < 0 ? 0 : (j >= ny ? ny - 1 : j);
    }
    return q[j * nx + i];
}

void or_step_scalar_2d(const or_map* ppx, const or_map* pmx, const or_map* ppy, const or_map* pmy,
                       int boundary, int64_t nx, int64_t ny, const int64_t* q, int64_t* out)
{
    #pragma omp parallel for schedule(static) if (nx * ny >= 32768)
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
            int64_t c = q[j * nx + i];
            int64_t Fxr = or_phi(ppx, c) + or_phi(pmx, at2(q, boundary, nx, ny, i + 1, j));
            int64_t Fxl = or_phi(ppx, at2(q, boundary, nx, ny, i - 1, j)) + or_phi(pmx, c);
            int64_t Fyr = or_phi(ppy, c) + or_phi(pmy, at2(q, boundary, nx, ny, i, j + 1));
            int64_t Fyl = or_phi(ppy, at2(q, boundary, nx, ny, i, j - 1)) + or_phi(pmy, c);
            out[j * nx + i] = c - (Fxr - Fxl) - (Fyr - Fyl);
        }
}

void or_run_scalar_2d(const or_map* ppx, const or_map* pmx, const or_map* ppy, const or_map* pmy,
                      int boundary, int64_t nx, int64_t ny, int64_t* q, int64_t nsteps,
                      int nthreads)
{
    set_threads(nthreads);
    const size_t N = (size_t)(nx * ny);
    int64_t* a = q;
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * N);
    for (int64_t s = 0; s < nsteps; ++s) {
        or_step_scalar_2d(ppx, pmx, ppy, pmy, boundary, nx, ny, a, b);
        int64_t* t = a; a = b; b = t;
    }
    if (a != q) { memcpy(q, a, sizeof(int64_t) * N); b = a; }
    free(b);
}

/* d = 3 (Thm P:364-401, Eq. nd_transfer_rule with d = 3), unsplit:
 *   q'_{i,j,k} = q - sum_{m = x,y,z} (F_{+e_m} - F_{-e_m}),
 *   F_{i+1/2 e_m} = phi+_m(q_i) + phi-_m(q_{i+e_m}),  all on q^n.
 * Layout q[(k * ny + j) * nx + i] (x fastest).  Boundaries per direction as in 1D. */
static int64_t wrap3(int boundary, int64_t i, int64_t n)
{
    if (boundary == OR_PERIODIC) return (i % n + n) % n;
    return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

void or_step_scalar_3d(const or_map* const* maps, int boundary, int64_t nx, int64_t ny,
                       int64_t nz, const int64_t* q, int64_t* out)
{
    /* maps = {phi+_x, phi-_x, phi+_y, phi-_y, phi+_z, phi-_z} */
    #pragma omp parallel for schedule(static) if (nx * ny * nz >= 32768)
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t c = q[(k * ny + j) * nx + i];
                const int64_t xp = q[(k * ny + j) * nx + wrap3(boundary, i + 1, nx)];
                const int64_t xm = q[(k * ny + j) * nx + wrap3(boundary, i - 1, nx)];
                const int64_t yp = q[(k * ny + wrap3(boundary, j + 1, ny)) * nx + i];
                const int64_t ym = q[(k * ny + wrap3(boundary, j - 1, ny)) * nx + i];
                const int64_t zp = q[(wrap3(boundary, k + 1, nz) * ny + j) * nx + i];
                const int64_t zm = q[(wrap3(boundary, k - 1, nz) * ny + j) * nx + i];
                const int64_t Fxr = or_phi(maps[0], c) + or_phi(maps[1], xp);
                const int64_t Fxl = or_phi(maps[0], xm) + or_phi(maps[1], c);
                const int64_t Fyr = or_phi(maps[2], c) + or_phi(maps[3], yp);
                const int64_t Fyl = or_phi(maps[2], ym) + or_phi(maps[3], c);
                const int64_t Fzr = or_phi(maps[4], c) + or_phi(maps[5], zp);
                const int64_t Fzl = or_phi(maps[4], zm) + or_phi(maps[5], c);
                out[(k * ny + j) * nx + i] = c - (Fxr - Fxl) - (Fyr - Fyl) - (Fzr - Fzl);
            }
}

void or_run_scalar_3d(const or_map* const* maps, int boundary, int64_t nx, int64_t ny, int64_t nz,
                      int64_t* q, int64_t nsteps, int nthreads)
{
    set_threads(nthreads);
    const size_t N = (size_t)(nx * ny * nz);
    int64_t* a = q;
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * N);
    for (int64_t s = 0; s < nsteps; ++s) {
        or_step_scalar_3d(maps, boundary, nx, ny, nz, a, b);
        int64_t* t = a; a = b; b = t;
    }
    if (a != q) { memcpy(q, a, sizeof(int64_t) * N); b = a; }
    free(b);
}

/* ---- 4. reconstruction ---------------------------------------------------- */
void or_observe(double delta, const int64_t* q, double* u, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) u[i] = delta * (double)q[i];
}

/* ---- 5. Euler system: quantised Roe transfer ------------------------------ */
/* Every statement below is one IEEE binary64 operation (+ - * / sqrt, all
 * correctly rounded), in the order of DESIGN.md reading R-ROE-2 (SURVEY
 * §8(c)-C2 with the divisions by rho, d and a^2 re-pinned as one reciprocal
 * each, multiplied in; the paper does not fix the arithmetic).
 * Compiled with -ffp-contract=off, so no FMA contraction or reassociation. */

typedef struct {
    double rho, m, E, u, p, H, r, f0, f1, f2;
} or_side;

static void or_roe_side_d(double g1, double rho, double m, double E, or_side* s)
{
    double irho = 1.0 / rho;
    double u = m * irho;
    double mu = m * u;
    double half_mu = 0.5 * mu;
    double e_int = E - half_mu;
    double p = g1 * e_int;
    double Ep = E + p;
    double H = Ep * irho;
    double r = sqrt(rho);
    s->rho = rho; s->m = m; s->E = E; s->u = u; s->p = p; s->H = H; s->r = r;
    s->f0 = m;
    s->f1 = mu + p;
    s->f2 = u * Ep;
}

static void or_roe_side(double delta, double g1, const int64_t qc[3], or_side* s)
{
    or_roe_side_d(g1, delta * (double)qc[0], delta * (double)qc[1], delta * (double)qc[2], s);
}

/* round-half-away-from-zero of a double (reading A1): exact because
 * x - trunc(x) is exact in binary64. */
static int64_t or_rha_double(double x)
{
    double t = trunc(x);
    double d = x - t;
    if (fabs(d) >= 0.5) t += (x > 0) ? 1.0 : -1.0;
    return (int64_t)t;
}

static double or_harten(double l, double eps)
{
    double al = fabs(l);
    if (al >= eps) return al;
    double ll = l * l;
    double ee = eps * eps;
    double num = ll + ee;
    double den = 2.0 * eps;
    return num / den;
}

/* Roe flux F^c(L, R) of two physical states (R-ROE-2 operation order). */
static void or_roe_flux(double g1, const or_side* Lp, const or_side* Rp, double F[3])
{
    or_side L = *Lp, R = *Rp;
    double d = L.r + R.r;
    double id = 1.0 / d;
    double ru_l = L.r * L.u, ru_r = R.r * R.u;
    double ut = (ru_l + ru_r) * id;
    double rh_l = L.r * L.H, rh_r = R.r * R.H;
    double Ht = (rh_l + rh_r) * id;
    double rhot = L.r * R.r;
    double uu = ut * ut;
    double half_uu = 0.5 * uu;
    double a2 = g1 * (Ht - half_uu);
    double at = sqrt(a2);
    double drho = R.rho - L.rho;
    double du = R.u - L.u;
    double dp = R.p - L.p;
    double ra = rhot * at;
    double t = ra * du;
    double ia2 = 1.0 / a2;
    double h_ia2 = 0.5 * ia2;
    double al1 = (dp - t) * h_ia2;
    double al3 = (dp + t) * h_ia2;
    double dpa = dp * ia2;
    double al2 = drho - dpa;
    double l1 = ut - at;
    double l3 = ut + at;
    double eps = 0.05 * (fabs(ut) + at);
    double c1 = or_harten(l1, eps) * al1;
    double c2 = fabs(ut) * al2;
    double c3 = or_harten(l3, eps) * al3;
    double ua = ut * at;
    double r1[3] = {1.0, l1, Ht - ua};
    double r2[3] = {1.0, ut, half_uu};
    double r3[3] = {1.0, l3, Ht + ua};
    double fL[3] = {L.f0, L.f1, L.f2};
    double fR[3] = {R.f0, R.f1, R.f2};
    for (int c = 0; c < 3; ++c) {
        double w1 = c1 * r1[c];
        double w3 = c3 * r3[c];
        double w2 = c2 * r2[c];
        double D = (w1 + w3) + w2;
        double avg = 0.5 * (fL[c] + fR[c]);
        F[c] = avg - 0.5 * D;
    }
}

/* T^c(qL, qR) = RHA(fl(F^c_Roe(delta qL, delta qR) * s)), s = fl(dt/dx / delta). */
void or_roe_transfer(double delta, double s, double g1, const int64_t qL[3],
                     const int64_t qR[3], int64_t T[3])
{
    or_side L, R;
    double F[3];
    or_roe_side(delta, g1, qL, &L);
    or_roe_side(delta, g1, qR, &R);
    or_roe_flux(g1, &L, &R, F);
    for (int c = 0; c < 3; ++c) {
        double x = F[c] * s;
        T[c] = or_rha_double(x);
    }
}

/* One explicit step of the componentwise-quantised Euler system, SoA [3][N],
 * transmissive boundaries (ghost copies, reading A12). */
void or_step_euler(double delta, double s, double g1, int64_t N,
                   const int64_t* q, int64_t* out)
{
    #pragma omp parallel for schedule(static) if (N >= 32768)
    for (int64_t i = 0; i < N; ++i) {
        int64_t im = i > 0 ? i - 1 : 0;
        int64_t ip = i < N - 1 ? i + 1 : N - 1;
        int64_t qi[3] = {q[i], q[N + i], q[2 * N + i]};
        int64_t qm[3] = {q[im], q[N + im], q[2 * N + im]};
        int64_t qp[3] = {q[ip], q[N + ip], q[2 * N + ip]};
        int64_t Tl[3], Tr[3];
        or_roe_transfer(delta, s, g1, qm, qi, Tl);
        or_roe_transfer(delta, s, g1, qi, qp, Tr);
        for (int c = 0; c < 3; ++c)
            out[c * N + i] = qi[c] - (Tr[c] - Tl[c]);
    }
}

/* Density-only quantisation (the paper's Sod prototype; DESIGN.md
 * reading A9-D): cell state (q_rho int64, m double, E double) in SoA [3][N]
 * (components 1 and 2 stored as IEEE doubles).  rho = delta q_rho enters the
 * same Roe flux; the density moves by integer transfers T = RHA(fl(F^rho s)),
 * momentum and energy by the classical float64 update
 * m' = fl(m - fl(lam fl(F^m_{i+1/2} - F^m_{i-1/2}))) (likewise E), transmissive. */
static void or_side_mixed(double delta, double g1, const int64_t* q, int64_t N, int64_t i,
                          or_side* s)
{
    double m, E;
    memcpy(&m, &q[N + i], 8);
    memcpy(&E, &q[2 * N + i], 8);
    or_roe_side_d(g1, delta * (double)q[i], m, E, s);
}

void or_step_euler_density(double delta, double s, double lam, double g1, int64_t N,
                           const int64_t* q, int64_t* out)
{
    #pragma omp parallel for schedule(static) if (N >= 32768)
    for (int64_t i = 0; i < N; ++i) {
        int64_t im = i > 0 ? i - 1 : 0;
        int64_t ip = i < N - 1 ? i + 1 : N - 1;
        or_side Sm, Si, Sp;
        or_side_mixed(delta, g1, q, N, im, &Sm);
        or_side_mixed(delta, g1, q, N, i, &Si);
        or_side_mixed(delta, g1, q, N, ip, &Sp);
        double Fl[3], Fr[3];
        or_roe_flux(g1, &Sm, &Si, Fl);
        or_roe_flux(g1, &Si, &Sp, Fr);
        int64_t Tl = or_rha_double(Fl[0] * s), Tr = or_rha_double(Fr[0] * s);
        out[i] = q[i] - (Tr - Tl);
        double m, E;
        memcpy(&m, &q[N + i], 8);
        memcpy(&E, &q[2 * N + i], 8);
        double dm = Fr[1] - Fl[1];
        double dE = Fr[2] - Fl[2];
        double m2 = m - lam * dm;
        double E2 = E - lam * dE;
        memcpy(&out[N + i], &m2, 8);
        memcpy(&out[2 * N + i], &E2, 8);
    }
}

void or_run_euler_density(double delta, double s, double lam, double g1, int64_t N, int64_t* q,
                          int64_t nsteps, int nthreads)
{
    set_threads(nthreads);
    int64_t* a = q;
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)N);
    for (int64_t k = 0; k < nsteps; ++k) {
        or_step_euler_density(delta, s, lam, g1, N, a, b);
        int64_t* t = a; a = b; b = t;
    }
    if (a != q) { memcpy(q, a, sizeof(int64_t) * 3 * (size_t)N); b = a; }
    free(b);
}

void or_run_euler(double delta, double s, double g1, int64_t N, int64_t* q,
                  int64_t nsteps, int nthreads)
{
    set_threads(nthreads);
    int64_t* a = q;
    int64_t* b = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)N);
    for (int64_t k = 0; k < nsteps; ++k) {
        or_step_euler(delta, s, g1, N, a, b);
        int64_t* t = a; a = b; b = t;
    }
    if (a != q) { memcpy(q, a, sizeof(int64_t) * 3 * (size_t)N); b = a; }
    free(b);
}

int or_max_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
