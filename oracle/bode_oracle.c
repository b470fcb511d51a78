/*
 * bode_oracle.c -- TEST INFRASTRUCTURE ONLY (see bode_oracle.h).
 *
 * Plain-C restatement of the reference CPU path. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Compiled with -ffp-contract=off and no -march flags so every operation is
 * a single IEEE binary64 rounding in the reference's expression order, as in
 * the reference's own Release build (CMakeLists.txt:8-10, no -march=native).
 *
 * Third-party arithmetic on the path: glibc libm (pow, cbrt, sqrt, lround),
 * called exactly where the reference calls it.
 */
#define _GNU_SOURCE
#include "bode_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ */
/* problems.cpp                                                        */
/* ------------------------------------------------------------------ */

/* problems.cpp:158-163 */
uint64_t orc_splitmix64_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* problems.cpp:165-169 */
double orc_unit_symmetric_at(uint64_t seed, uint64_t k) {
    const double u01 = (double)(orc_splitmix64_at(seed, k) >> 11) * 0x1.0p-53;
    return 2.0 * u01 - 1.0;
}

/* problems.cpp:171-191 */
int orc_perturb(const double* base, int dim, double magnitude, uint64_t seed,
                int count, double* out) {
    if (count < 1 || dim < 1) return BODE_E_INVALID_SHAPE;
    if (!(magnitude >= 0.0 && magnitude <= 0.1)) return BODE_E_INVALID_SHAPE;
    for (int i = 0; i < count; ++i)
        for (int j = 0; j < dim; ++j) {
            const uint64_t k = (uint64_t)i * (uint64_t)dim + (uint64_t)j;
            const double u = orc_unit_symmetric_at(seed, k);
            out[(size_t)i + (size_t)count * (size_t)j] = base[j] * (1.0 + u * magnitude);
        }
    return BODE_OK;
}

/* problems.cpp:13-35 (Pleiades RHS, masses m_i = i + 1, i outer, j inner) */
static void rhs_pleiades(const double* w, double* out) {
    const double* x = w;
    const double* y = w + 7;
    for (int i = 0; i < 14; ++i) out[i] = w[14 + i];
    for (int i = 14; i < 28; ++i) out[i] = 0.0;
    for (int i = 0; i < 7; ++i) {
        for (int j = i + 1; j < 7; ++j) {
            const double dx = x[j] - x[i];
            const double dy = y[j] - y[i];
            const double r2 = dx * dx + dy * dy;
            const double invR3 = 1.0 / (r2 * sqrt(r2));
            const double mi = (double)(i + 1);
            const double mj = (double)(j + 1);
            out[14 + i] += mj * dx * invR3;
            out[21 + i] += mj * dy * invR3;
            out[14 + j] -= mi * dx * invR3;
            out[21 + j] -= mi * dy * invR3;
        }
    }
}

/* problems.cpp:100-109 (dx = 1/(n+1), invDx2 = 1/(dx*dx)) */
static void rhs_heat(int n, const double* u, double* out) {
    const double dx = 1.0 / (n + 1);
    const double invDx2 = 1.0 / (dx * dx);
    out[0] = (-2.0 * u[0] + u[1]) * invDx2;
    for (int i = 1; i + 1 < n; ++i) out[i] = (u[i - 1] - 2.0 * u[i] + u[i + 1]) * invDx2;
    out[n - 1] = (u[n - 2] - 2.0 * u[n - 1]) * invDx2;
}

void orc_rhs(const bode_problem_t* p, double t, const double* y, const double* g,
             double* out) {
    const int n = p->dim;
    switch (p->kind) {
        case BODE_PROBLEM_PLEIADES: rhs_pleiades(y, out); break;
        case BODE_PROBLEM_HEAT: rhs_heat(n, y, out); break;
        case BODE_PROBLEM_EXPDECAY: out[0] = -g[0] * y[0]; break; /* problems.cpp:138-139 */
        case BODE_PROBLEM_HARMONIC: /* problems.cpp:150-154 */
            out[0] = y[1];
            out[1] = -y[0];
            break;
        case BODE_PROBLEM_ZERO:
            for (int i = 0; i < n; ++i) out[i] = 0.0;
            break;
        case BODE_PROBLEM_RICCATI: out[0] = y[0] * y[0]; break;
        case BODE_PROBLEM_DIAG:
            for (int i = 0; i < n; ++i) out[i] = g[i] * y[i];
            break;
        case BODE_PROBLEM_CONST:
            for (int i = 0; i < n; ++i) out[i] = 1.0;
            break;
        case BODE_PROBLEM_SINT: out[0] = sin(t) * y[0]; break;
        default:
            for (int i = 0; i < n; ++i) out[i] = NAN;
            break;
    }
}

/* problems.cpp:117-122 */
double orc_heat_spectral_radius(int interiorPoints) {
    const double n = (double)interiorPoints;
    const double dx = 1.0 / (n + 1.0);
    const double s = sin(n * M_PI / (2.0 * (n + 1.0)));
    return 4.0 / (dx * dx) * s * s;
}

/* problems.cpp:124-132 */
void orc_heat_initial_condition(int n, double* u) {
    const double dx = 1.0 / (n + 1);
    for (int i = 0; i < n; ++i) {
        const double x = (i + 1) * dx;
        u[i] = 4.0 * x * (1.0 - x);
    }
}

/* problems.cpp:66-82 */
double orc_pleiades_energy(const double* w) {
    double kinetic = 0.0;
    for (int i = 0; i < 7; ++i) {
        const double m = (double)(i + 1);
        kinetic += 0.5 * m * (w[14 + i] * w[14 + i] + w[21 + i] * w[21 + i]);
    }
    double potential = 0.0;
    for (int i = 0; i < 7; ++i)
        for (int j = i + 1; j < 7; ++j) {
            const double dx = w[i] - w[j];
            const double dy = w[7 + i] - w[7 + j];
            potential -= (double)(i + 1) * (double)(j + 1) / sqrt(dx * dx + dy * dy);
        }
    return kinetic + potential;
}

/* problems.cpp:84-92 */
void orc_pleiades_momentum(const double* w, double out[2]) {
    double px = 0.0, py = 0.0;
    for (int i = 0; i < 7; ++i) {
        const double m = (double)(i + 1);
        px += m * w[14 + i];
        py += m * w[21 + i];
    }
    out[0] = px;
    out[1] = py;
}

/* ------------------------------------------------------------------ */
/* rkck.cpp                                                            */
/* ------------------------------------------------------------------ */

/* rkck.cpp:8-27 (Cash-Karp tableau, Table 1 of PAPER.md:86-103) */
static const double kA[6] = {0.0, 1.0 / 5.0, 3.0 / 10.0, 3.0 / 5.0, 1.0, 7.0 / 8.0};
static const double kB[6][5] = {
    {0.0, 0.0, 0.0, 0.0, 0.0},
    {1.0 / 5.0, 0.0, 0.0, 0.0, 0.0},
    {3.0 / 40.0, 9.0 / 40.0, 0.0, 0.0, 0.0},
    {3.0 / 10.0, -9.0 / 10.0, 6.0 / 5.0, 0.0, 0.0},
    {-11.0 / 54.0, 5.0 / 2.0, -70.0 / 27.0, 35.0 / 27.0, 0.0},
    {1631.0 / 55296.0, 175.0 / 512.0, 575.0 / 13824.0, 44275.0 / 110592.0, 253.0 / 4096.0}};
static const double kC[6] = {37.0 / 378.0, 0.0, 250.0 / 621.0, 125.0 / 594.0, 0.0,
                             512.0 / 1771.0};
static const double kCs[6] = {2825.0 / 27648.0, 0.0, 18575.0 / 48384.0,
                              13525.0 / 55296.0, 277.0 / 14336.0, 1.0 / 4.0};

#define ORC_MAXDIM 4096

/* rkck.cpp:34-78 */
void orc_rkck_step(const bode_problem_t* p, double t, const double* y,
                   const double* g, const double* f0, double h, double* yNext,
                   double* yErr) {
    const int n = p->dim;
    double* buf = (double*)malloc(sizeof(double) * 6 * (size_t)n);
    double *ytemp = buf, *k2 = buf + n, *k3 = buf + 2 * n, *k4 = buf + 3 * n,
           *k5 = buf + 4 * n, *k6 = buf + 5 * n;
    for (int i = 0; i < n; ++i) ytemp[i] = y[i] + h * kB[1][0] * f0[i];
    orc_rhs(p, t + kA[1] * h, ytemp, g, k2);
    for (int i = 0; i < n; ++i) ytemp[i] = y[i] + h * (kB[2][0] * f0[i] + kB[2][1] * k2[i]);
    orc_rhs(p, t + kA[2] * h, ytemp, g, k3);
    for (int i = 0; i < n; ++i)
        ytemp[i] = y[i] + h * (kB[3][0] * f0[i] + kB[3][1] * k2[i] + kB[3][2] * k3[i]);
    orc_rhs(p, t + kA[3] * h, ytemp, g, k4);
    for (int i = 0; i < n; ++i)
        ytemp[i] = y[i] + h * (kB[4][0] * f0[i] + kB[4][1] * k2[i] + kB[4][2] * k3[i] +
                               kB[4][3] * k4[i]);
    orc_rhs(p, t + kA[4] * h, ytemp, g, k5);
    for (int i = 0; i < n; ++i)
        ytemp[i] = y[i] + h * (kB[5][0] * f0[i] + kB[5][1] * k2[i] + kB[5][2] * k3[i] +
                               kB[5][3] * k4[i] + kB[5][4] * k5[i]);
    orc_rhs(p, t + kA[5] * h, ytemp, g, k6);
    /* rkck.cpp:67-77: c2 = c5 = 0, d = c - c* */
    const double c1 = kC[0], c3 = kC[2], c4 = kC[3], c6 = kC[5];
    const double d1 = kC[0] - kCs[0];
    const double d3 = kC[2] - kCs[2];
    const double d4 = kC[3] - kCs[3];
    const double d5 = kC[4] - kCs[4];
    const double d6 = kC[5] - kCs[5];
    for (int i = 0; i < n; ++i) {
        yNext[i] = y[i] + h * (c1 * f0[i] + c3 * k3[i] + c4 * k4[i] + c6 * k6[i]);
        yErr[i] = h * (d1 * f0[i] + d3 * k3[i] + d4 * k4[i] + d5 * k5[i] + d6 * k6[i]);
    }
    free(buf);
}

/* rkck.cpp:88-98 */
void orc_rkck_error_norm(int n, const double* y, const double* f0,
                         const double* yErr, double h, double eps, double tiny,
                         double* errOut, int* nanFlag) {
    double err = 0.0;
    int nan = 0;
    for (int i = 0; i < n; ++i) {
        if (!isfinite(yErr[i])) nan = 1;
        err = fmax(err, fabs(yErr[i] / (fabs(y[i]) + fabs(h * f0[i]) + tiny)));
    }
    *errOut = err / eps;
    *nanFlag = nan;
}

/* rkck.cpp:100-113 */
void orc_rkck_adjust_step(double h, double err, int nanFlag, double hMin,
                          double hMax, const bode_tol_t* tol, int* accepted,
                          double* hNew) {
    if (err > 1.0 || !isfinite(err) || nanFlag) {
        *hNew = (!isfinite(err) || nanFlag)
                    ? tol->p1 * h
                    : fmax(tol->safety * h * pow(err, tol->pshrnk), tol->p1 * h);
        *accepted = 0;
        return;
    }
    double hn = (err > tol->errcon) ? tol->safety * h * pow(err, tol->pgrow) : 5.0 * h;
    *hNew = fmax(hMin, fmin(hMax, hn));
    *accepted = 1;
}

static void stats_init(bode_stats_t* st) {
    memset(st, 0, sizeof(*st));
    st->h_min_seen = INFINITY;
    st->h_max_seen = 0.0;
}

/* ode_problem.hpp:66-70 */
static void stats_record_accepted(bode_stats_t* st, double h) {
    ++st->steps_accepted;
    st->h_min_seen = fmin(st->h_min_seen, h);
    st->h_max_seen = fmax(st->h_max_seen, h);
}

/* ode_problem.hpp:72-80 */
static void stats_merge(bode_stats_t* a, const bode_stats_t* b) {
    a->steps_accepted += b->steps_accepted;
    a->steps_rejected += b->steps_rejected;
    a->rhs_evals += b->rhs_evals;
    a->spec_rad_evals += b->spec_rad_evals;
    a->stages_total += b->stages_total;
    a->h_min_seen = fmin(a->h_min_seen, b->h_min_seen);
    a->h_max_seen = fmax(a->h_max_seen, b->h_max_seen);
    a->underflow = a->underflow || b->underflow;
}

/* rkck.cpp:115-159 */
int orc_rkck_driver(const bode_problem_t* p, double t, double tEnd, double* y,
                    const double* g, const bode_tol_t* tol, bode_stats_t* st,
                    orc_observer_fn obs, void* user) {
    if (!(tEnd > t)) return BODE_E_INVALID_INTERVAL;
    const int n = p->dim;
    double* buf = (double*)malloc(sizeof(double) * 3 * (size_t)n);
    double *f0 = buf, *yNext = buf + n, *yErr = buf + 2 * n;
    const double hMax = fabs(tEnd - t);
    const double hMin = tol->h_min_floor;
    double h = 0.5 * fabs(tEnd - t);
    stats_init(st);
    int haveF = 0;
    while (tEnd - t > tol->uround * fabs(tEnd)) {
        h = fmin(tEnd - t, h);
        if (!haveF) {
            orc_rhs(p, t, y, g, f0);
            ++st->rhs_evals;
            haveF = 1;
        }
        orc_rkck_step(p, t, y, g, f0, h, yNext, yErr);
        st->rhs_evals += 5;
        st->stages_total += 6;
        double err;
        int nanFlag, accepted;
        double hNew;
        orc_rkck_error_norm(n, y, f0, yErr, h, tol->eps, tol->tiny, &err, &nanFlag);
        orc_rkck_adjust_step(h, err, nanFlag, hMin, hMax, tol, &accepted, &hNew);
        if (obs) obs(t, h, 6, err, accepted, user);
        if (accepted) {
            t += h;
            stats_record_accepted(st, h);
            memcpy(y, yNext, sizeof(double) * (size_t)n);
            haveF = 0;
            h = hNew;
        } else {
            ++st->steps_rejected;
            if (hNew < tol->h_min_floor) {
                st->underflow = 1;
                break;
            }
            h = hNew;
        }
    }
    free(buf);
    return BODE_OK;
}

/* rkck.cpp:168-181 */
void orc_rkck_integrate_fixed(const bode_problem_t* p, double t0, double tEnd,
                              long numSteps, double* y, const double* g) {
    const int n = p->dim;
    double* buf = (double*)malloc(sizeof(double) * 3 * (size_t)n);
    double *f0 = buf, *yNext = buf + n, *yErr = buf + 2 * n;
    const double h = (tEnd - t0) / (double)numSteps;
    for (long k = 0; k < numSteps; ++k) {
        const double t = t0 + (double)k * h;
        orc_rhs(p, t, y, g, f0);
        orc_rkck_step(p, t, y, g, f0, h, yNext, yErr);
        memcpy(y, yNext, sizeof(double) * (size_t)n);
    }
    free(buf);
}

/* ------------------------------------------------------------------ */
/* rkc.cpp                                                             */
/* ------------------------------------------------------------------ */

/* rkc.cpp:10-27 */
void orc_chebyshev_eval(int degree, double x, double out[3]) {
    if (degree <= 0) { out[0] = 1.0; out[1] = 0.0; out[2] = 0.0; return; }
    if (degree == 1) { out[0] = x; out[1] = 1.0; out[2] = 0.0; return; }
    double Tm2 = 1.0, Tm1 = x, dm2 = 0.0, dm1 = 1.0, ddm2 = 0.0, ddm1 = 0.0;
    for (int j = 2; j <= degree; ++j) {
        const double T = 2.0 * x * Tm1 - Tm2;
        const double d = 2.0 * Tm1 + 2.0 * x * dm1 - dm2;
        const double dd = 4.0 * dm1 + 2.0 * x * ddm1 - ddm2;
        Tm2 = Tm1; Tm1 = T;
        dm2 = dm1; dm1 = d;
        ddm2 = ddm1; ddm1 = dd;
    }
    out[0] = Tm1; out[1] = dm1; out[2] = ddm1;
}

/* rkc.cpp:29-69 */
int orc_rkc_coefficients(int stages, double kappa, double* omega0p, double* omega1p,
                         double* mu, double* nu, double* muTilde, double* gammaTilde,
                         double* b, double* a, double* c) {
    if (stages < 2) return BODE_E_INVALID_STAGE_COUNT;
    const double omega0 = 1.0 + kappa / ((double)stages * stages);
    double* T = (double*)malloc(sizeof(double) * 3 * (size_t)(stages + 1));
    for (int j = 0; j <= stages; ++j) orc_chebyshev_eval(j, omega0, T + 3 * j);
    const double omega1 = T[3 * stages + 1] / T[3 * stages + 2];
    for (int j = 0; j <= stages; ++j)
        b[j] = a[j] = c[j] = mu[j] = nu[j] = muTilde[j] = gammaTilde[j] = 0.0;
    for (int j = 2; j <= stages; ++j) b[j] = T[3 * j + 2] / (T[3 * j + 1] * T[3 * j + 1]);
    b[0] = b[2];
    b[1] = 1.0 / omega0;
    for (int j = 0; j <= stages; ++j) a[j] = 1.0 - b[j] * T[3 * j];
    muTilde[1] = b[1] * omega1;
    for (int j = 2; j <= stages; ++j) {
        mu[j] = 2.0 * b[j] * omega0 / b[j - 1];
        nu[j] = -b[j] / b[j - 2];
        muTilde[j] = 2.0 * b[j] * omega1 / b[j - 1];
        gammaTilde[j] = -a[j - 1] * muTilde[j];
    }
    for (int j = 2; j < stages; ++j) c[j] = omega1 * T[3 * j + 2] / T[3 * j + 1];
    c[stages] = 1.0;
    c[1] = c[2] / (4.0 * omega0);
    *omega0p = omega0;
    *omega1p = omega1;
    free(T);
    return BODE_OK;
}

typedef struct {
    int stages;
    double kappa;
    double *mu, *nu, *muTilde, *gammaTilde, *b, *a, *c;
    int cap;
} coef_cache_t;

/* rkc.cpp:76-80 (coefficientsFor cache) */
static int coef_for(coef_cache_t* cc, int stages, double kappa) {
    if (cc->stages == stages && cc->kappa == kappa) return BODE_OK;
    if (stages + 1 > cc->cap) {
        free(cc->mu);
        cc->cap = stages + 1;
        cc->mu = (double*)malloc(sizeof(double) * 7 * (size_t)cc->cap);
    }
    double* base = cc->mu;
    cc->nu = base + cc->cap;
    cc->muTilde = base + 2 * cc->cap;
    cc->gammaTilde = base + 3 * cc->cap;
    cc->b = base + 4 * cc->cap;
    cc->a = base + 5 * cc->cap;
    cc->c = base + 6 * cc->cap;
    double o0, o1;
    int rc = orc_rkc_coefficients(stages, kappa, &o0, &o1, cc->mu, cc->nu, cc->muTilde,
                                  cc->gammaTilde, cc->b, cc->a, cc->c);
    cc->stages = stages;
    cc->kappa = kappa;
    return rc;
}

/* rkc.cpp:82-117 */
static void rkc_step_cf(const bode_problem_t* p, double t, const double* y,
                        const double* g, const double* f0, double h,
                        const coef_cache_t* cf, double* yNext, double* scratch) {
    const int n = p->dim;
    const int stages = cf->stages;
    double* wjm1 = scratch;
    double* wjm2 = scratch + n;
    double* fstage = scratch + 2 * n;
    const double mu1h = cf->muTilde[1] * h;
    for (int i = 0; i < n; ++i) wjm1[i] = y[i] + mu1h * f0[i];
    int prevIsY = 1;
    for (int j = 2; j <= stages; ++j) {
        orc_rhs(p, t + cf->c[j - 1] * h, wjm1, g, fstage);
        const double muj = cf->mu[j];
        const double nuj = cf->nu[j];
        const double mujh = cf->muTilde[j] * h;
        const double gjh = cf->gammaTilde[j] * h;
        double* out = wjm2;
        if (prevIsY) {
            for (int i = 0; i < n; ++i)
                out[i] = y[i] + muj * (wjm1[i] - y[i]) + mujh * fstage[i] + gjh * f0[i];
            prevIsY = 0;
        } else {
            for (int i = 0; i < n; ++i)
                out[i] = y[i] + muj * (wjm1[i] - y[i]) + nuj * (wjm2[i] - y[i]) +
                         mujh * fstage[i] + gjh * f0[i];
        }
        double* tmp = wjm1;
        wjm1 = wjm2;
        wjm2 = tmp;
    }
    memcpy(yNext, wjm1, sizeof(double) * (size_t)n);
}

int orc_rkc_step(const bode_problem_t* p, double t, const double* y,
                 const double* g, const double* f0, double h, int stages,
                 double kappa, double* yNext) {
    coef_cache_t cc = {0};
    cc.stages = -1;
    int rc = coef_for(&cc, stages, kappa);
    if (rc != BODE_OK) { free(cc.mu); return rc; }
    double* scratch = (double*)malloc(sizeof(double) * 3 * (size_t)p->dim);
    rkc_step_cf(p, t, y, g, f0, h, &cc, yNext, scratch);
    free(scratch);
    free(cc.mu);
    return BODE_OK;
}

/* rkc.cpp:119-129 */
double orc_rkc_error_norm(int n, const double* yOld, const double* yNew,
                          const double* fOld, const double* fNew, double h,
                          double absTol, double relTol) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        double est = 0.8 * (yOld[i] - yNew[i]) + 0.4 * h * (fOld[i] + fNew[i]);
        est /= absTol + relTol * fmax(fabs(yOld[i]), fabs(yNew[i]));
        sum += est * est;
    }
    return sqrt(sum / (double)n);
}

/* rkc.cpp:131-144 */
void orc_rkc_stage_count(double h, double sigma, double relTol, double uround,
                         int* stagesOut, double* hOut) {
    long mMax = lround(sqrt(relTol / (10.0 * uround)));
    if (mMax < 2) mMax = 2;
    const double raw = sqrt(1.54 * h * sigma + 1.0);
    long s = raw < (double)mMax ? 1 + (long)raw : mMax + 1;
    double ho = h;
    if (s > mMax) {
        s = mMax;
        ho = ((double)s * (double)s - 1.0) / (1.54 * sigma);
    }
    *stagesOut = (int)s;
    *hOut = ho;
}

/* rkc.cpp:146-171 */
void orc_rkc_initial_step(const bode_problem_t* p, double t, const double* y,
                          const double* g, const double* f0, double sigma,
                          double hMax, double hMin, const bode_tol_t* tol,
                          double* hOut, double* errOut) {
    const int n = p->dim;
    double* w1 = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    double* fstage = w1 + n;
    double h = hMax;
    if (sigma * h > 1.0) h = 1.0 / sigma;
    h = fmax(h, hMin);
    for (int i = 0; i < n; ++i) w1[i] = y[i] + h * f0[i];
    orc_rhs(p, t + h, w1, g, fstage);
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        const double est = (fstage[i] - f0[i]) / (tol->abs_tol + tol->rel_tol * fabs(y[i]));
        sum += est * est;
    }
    const double err = h * sqrt(sum / (double)n);
    if (0.1 * h < hMax * sqrt(err))
        h = fmax(0.1 * h / sqrt(err), hMin);
    else
        h = hMax;
    *hOut = h;
    *errOut = err;
    free(w1);
}

/* rkc.cpp:173-187 */
double orc_rkc_next_step_accepted(double err, double errOld, double h, double hOld,
                                  int firstAccepted, double hMin, double hMax) {
    double fac = 10.0;
    if (firstAccepted) {
        const double t2 = cbrt(err);
        if (0.8 < fac * t2) fac = 0.8 / t2;
    } else {
        const double t1 = 0.8 * h * cbrt(errOld);
        const double cb = cbrt(err);
        const double t2 = hOld * cb * cb;
        if (t1 < fac * t2) fac = t1 / t2;
    }
    const double hNew = h * fmax(0.1, fac);
    return fmax(hMin, fmin(hMax, hNew));
}

/* rkc.cpp:189-191 */
double orc_rkc_next_step_rejected(double err, double h) { return 0.8 * h / cbrt(err); }

/* spectral_radius.cpp:11-15 */
static double norm2(int n, const double* v) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* spectral_radius.cpp:17-85 */
int orc_power_method(const bode_problem_t* p, double t, const double* y,
                     const double* g, const double* f0, double hMax,
                     const double* vWarm, double* sigmaOut, double* eigvec,
                     int* iterations, int* converged) {
    const int n = p->dim;
    const int kItMax = 50;
    const double kUround = 2.22e-16;
    const double sqrtU = sqrt(kUround);
    const double small = 1.0 / hMax;
    double* v = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    double* fv = v + n;
    memcpy(v, vWarm, sizeof(double) * (size_t)n);
    const double nrmY = norm2(n, y);
    const double nrmV = norm2(n, v);
    double dynrm;
    if (nrmY != 0.0 && nrmV != 0.0) {
        dynrm = nrmY * sqrtU;
        for (int i = 0; i < n; ++i) v[i] = y[i] + v[i] * (dynrm / nrmV);
    } else if (nrmY != 0.0) {
        dynrm = nrmY * sqrtU;
        for (int i = 0; i < n; ++i) v[i] = y[i] * (1.0 + sqrtU);
    } else if (nrmV != 0.0) {
        dynrm = kUround;
        for (int i = 0; i < n; ++i) v[i] *= dynrm / nrmV;
    } else {
        dynrm = kUround;
        for (int i = 0; i < n; ++i) v[i] = kUround;
    }
    int iters = 0, conv = 0;
    double sigma = 0.0;
    for (int iter = 1; iter <= kItMax; ++iter) {
        orc_rhs(p, t, v, g, fv);
        iters = iter;
        double diffNrm = 0.0;
        for (int i = 0; i < n; ++i) {
            const double d = fv[i] - f0[i];
            diffNrm += d * d;
        }
        diffNrm = sqrt(diffNrm);
        const double sigmaOld = sigma;
        sigma = diffNrm / dynrm;
        if (iter >= 2 && fabs(sigma - sigmaOld) <= fmax(sigma, small) * 0.01) {
            conv = 1;
            break;
        }
        if (diffNrm != 0.0) {
            for (int i = 0; i < n; ++i) v[i] = y[i] + (fv[i] - f0[i]) * (dynrm / diffNrm);
        } else {
            const int ind = iter % n;
            v[ind] = y[ind] - (v[ind] - y[ind]);
        }
    }
    *sigmaOut = 1.2 * sigma;
    for (int i = 0; i < n; ++i) eigvec[i] = v[i] - y[i];
    *iterations = iters;
    *converged = conv;
    free(v);
    return BODE_OK;
}

/* rkc.cpp:193-281 */
static int rkc_driver_impl(const bode_problem_t* p, double t, double tEnd, double* y,
                           const double* g, const bode_tol_t* tol, bode_stats_t* st,
                           orc_observer_fn obs, void* user, coef_cache_t* cc) {
    if (!(tEnd > t)) return BODE_E_INVALID_INTERVAL;
    const int n = p->dim;
    double* buf = (double*)malloc(sizeof(double) * 7 * (size_t)n);
    double *f0 = buf, *ytrial = buf + n, *ftrial = buf + 2 * n, *eig = buf + 3 * n,
           *scratch = buf + 4 * n;
    /* Workspace::reset (rkc.hpp:57-60): restart every invocation */
    double wsErrOld = 0.0, wsHOld = 0.0, wsH = 0.0, wsSpecRad = 0.0;
    const double hMax = fabs(tEnd - t);
    stats_init(st);
    long numStep = 0;
    orc_rhs(p, t, y, g, f0);
    ++st->rhs_evals;
    memcpy(eig, f0, sizeof(double) * (size_t)n);

#define ESTIMATE_SPEC_RAD()                                                        \
    do {                                                                           \
        double sig_;                                                               \
        int it_, cv_;                                                              \
        orc_power_method(p, t, y, g, f0, hMax, eig, &sig_, eig, &it_, &cv_);       \
        wsSpecRad = sig_;                                                          \
        ++st->spec_rad_evals;                                                      \
        st->rhs_evals += it_;                                                      \
    } while (0)

    while (tEnd - t > tol->uround * fabs(tEnd)) {
        const double hMin = 10.0 * tol->uround * fmax(fabs(t), hMax);
        if (1.1 * wsH >= fabs(tEnd - t)) wsH = fabs(tEnd - t);
        if (numStep % 25 == 0) ESTIMATE_SPEC_RAD();
        if (wsH < tol->uround) {
            double hi, ei;
            orc_rkc_initial_step(p, t, y, g, f0, wsSpecRad, hMax, hMin, tol, &hi, &ei);
            ++st->rhs_evals;
            wsH = hi;
        }
        const double sigma = isfinite(wsSpecRad) ? wsSpecRad : 0.0;
        int stages;
        double hs;
        orc_rkc_stage_count(wsH, sigma, tol->rel_tol, tol->uround, &stages, &hs);
        wsH = hs;
        coef_for(cc, stages, tol->kappa);
        rkc_step_cf(p, t, y, g, f0, wsH, cc, ytrial, scratch);
        st->rhs_evals += stages - 1;
        st->stages_total += stages;
        orc_rhs(p, t + wsH, ytrial, g, ftrial);
        ++st->rhs_evals;
        const double err =
            orc_rkc_error_norm(n, y, ytrial, f0, ftrial, wsH, tol->abs_tol, tol->rel_tol);
        const int accepted = err <= 1.0;
        if (obs) obs(t, wsH, stages, err, accepted, user);
        if (!accepted) {
            ++st->steps_rejected;
            const double hNew =
                isfinite(err) ? orc_rkc_next_step_rejected(err, wsH) : tol->p1 * wsH;
            ESTIMATE_SPEC_RAD();
            if (hNew < hMin) {
                st->underflow = 1;
                break;
            }
            wsH = hNew;
        } else {
            t += wsH;
            ++numStep;
            stats_record_accepted(st, wsH);
            const int firstAccepted = wsHOld < tol->uround;
            const double hNew = orc_rkc_next_step_accepted(err, wsErrOld, wsH, wsHOld,
                                                           firstAccepted, hMin, hMax);
            wsErrOld = fmax(err, tol->uround);
            wsHOld = wsH;
            memcpy(y, ytrial, sizeof(double) * (size_t)n);
            double* tmp = f0; /* FSAL swap f0 <-> ftrial (rkc.cpp:276) */
            f0 = ftrial;
            ftrial = tmp;
            wsH = hNew;
        }
    }
#undef ESTIMATE_SPEC_RAD
    free(buf);
    return BODE_OK;
}

int orc_rkc_driver(const bode_problem_t* p, double t, double tEnd, double* y,
                   const double* g, const bode_tol_t* tol, bode_stats_t* st,
                   orc_observer_fn obs, void* user) {
    coef_cache_t cc = {0};
    cc.stages = -1;
    int rc = rkc_driver_impl(p, t, tEnd, y, g, tol, st, obs, user, &cc);
    free(cc.mu);
    return rc;
}

/* rkc.cpp:290-306 */
void orc_rkc_integrate_fixed(const bode_problem_t* p, double t0, double tEnd,
                             long numSteps, int stages, double kappa, double* y,
                             const double* g) {
    const int n = p->dim;
    coef_cache_t cc = {0};
    cc.stages = -1;
    coef_for(&cc, stages, kappa);
    double* buf = (double*)malloc(sizeof(double) * 5 * (size_t)n);
    double *f0 = buf, *ynext = buf + n, *scratch = buf + 2 * n;
    const double h = (tEnd - t0) / (double)numSteps;
    for (long k = 0; k < numSteps; ++k) {
        const double t = t0 + (double)k * h;
        orc_rhs(p, t, y, g, f0);
        rkc_step_cf(p, t, y, g, f0, h, &cc, ynext, scratch);
        memcpy(y, ynext, sizeof(double) * (size_t)n);
    }
    free(buf);
    free(cc.mu);
}

/* ------------------------------------------------------------------ */
/* batch_driver.cpp                                                    */
/* ------------------------------------------------------------------ */

static int tol_validate(const bode_tol_t* tol) { /* ode_problem.hpp:46-53 */
    if (!(tol->eps > 0.0 && tol->abs_tol > 0.0 && tol->rel_tol > 0.0))
        return BODE_E_INVALID_SHAPE;
    if (!(tol->safety > 0.0 && tol->safety < 1.0) || !(tol->p1 > 0.0 && tol->p1 < 1.0))
        return BODE_E_INVALID_SHAPE;
    if (!(tol->uround > 0.0 && tol->tiny > 0.0 && tol->h_min_floor > 0.0 &&
          tol->kappa >= 0.0))
        return BODE_E_INVALID_SHAPE;
    return BODE_OK;
}

typedef struct {
    const bode_problem_t* p;
    int solver;
    double t, tNext;
    int64_t num, begin, end;
    double* y;
    const double* g;
    const bode_tol_t* tol;
    bode_stats_t* stats;
    int merge;
} chunk_t;

/* batch_driver.cpp:17-35: gather, drive, scatter per system */
static void* integrate_chunk(void* arg) {
    chunk_t* c = (chunk_t*)arg;
    const int n = c->p->dim, np = c->p->param_dim;
    double* yl = (double*)malloc(sizeof(double) * (size_t)(n + np + 1));
    double* gl = yl + n;
    coef_cache_t cc = {0};
    cc.stages = -1;
    for (int64_t i = c->begin; i < c->end; ++i) {
        for (int j = 0; j < n; ++j) yl[j] = c->y[i + c->num * j];
        for (int j = 0; j < np; ++j) gl[j] = c->g[i + c->num * j];
        bode_stats_t st;
        if (c->solver == BODE_SOLVER_RKCK)
            orc_rkck_driver(c->p, c->t, c->tNext, yl, gl, c->tol, &st, NULL, NULL);
        else
            rkc_driver_impl(c->p, c->t, c->tNext, yl, gl, c->tol, &st, NULL, NULL, &cc);
        for (int j = 0; j < n; ++j) c->y[i + c->num * j] = yl[j];
        if (c->stats) {
            if (c->merge)
                stats_merge(&c->stats[i], &st);
            else
                c->stats[i] = st;
        }
    }
    free(cc.mu);
    free(yl);
    return NULL;
}

static int batch_impl(const bode_problem_t* p, int solver, double t, double tNext,
                      int64_t num, double* y, const double* g, const bode_tol_t* tol,
                      bode_stats_t* stats, int threads, int merge) {
    if (!(tNext > t)) return BODE_E_INVALID_INTERVAL;
    if (num < 1 || p->dim < 1 || p->param_dim < 0) return BODE_E_INVALID_SHAPE;
    if (tol_validate(tol) != BODE_OK) return BODE_E_INVALID_SHAPE;
    if (threads < 1) return BODE_E_INVALID_SHAPE;
    if (threads > num) threads = (int)num;
    chunk_t* chunks = (chunk_t*)malloc(sizeof(chunk_t) * (size_t)threads);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    /* batch_driver.cpp:68-73: contiguous static partition */
    const int64_t base = num / threads, rem = num % threads;
    int64_t begin = 0;
    for (int w = 0; w < threads; ++w) {
        const int64_t len = base + (w < rem ? 1 : 0);
        chunk_t c = {p, solver, t, tNext, num, begin, begin + len, y, g, tol, stats, merge};
        chunks[w] = c;
        begin += len;
    }
    if (threads == 1) {
        integrate_chunk(&chunks[0]);
    } else {
        for (int w = 0; w < threads; ++w) pthread_create(&th[w], NULL, integrate_chunk, &chunks[w]);
        for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
    }
    free(th);
    free(chunks);
    return BODE_OK;
}

/* batch_driver.cpp:39-88 */
int orc_integrate_batch(const bode_problem_t* p, int solver, double t, double tNext,
                        int64_t num, double* y, const double* g, const bode_tol_t* tol,
                        bode_stats_t* stats, int threads) {
    return batch_impl(p, solver, t, tNext, num, y, g, tol, stats, threads, 0);
}

/* batch_driver.cpp:90-116 */
int orc_outer_loop(const bode_problem_t* p, int solver, double t0, double tEnd,
                   double hOuter, int64_t num, double* y, const double* g,
                   const bode_tol_t* tol, bode_stats_t* stats, int threads,
                   int* outerSteps) {
    if (!(tEnd > t0)) return BODE_E_INVALID_INTERVAL;
    if (!(hOuter > 0.0)) return BODE_E_INVALID_INTERVAL;
    const double ratio = (tEnd - t0) / hOuter;
    long nWindows = (long)ceil(ratio - 1e-9);
    if (nWindows < 1) nWindows = 1;
    if (stats)
        for (int64_t i = 0; i < num; ++i) stats_init(&stats[i]);
    double t = t0;
    int steps = 0;
    for (long k = 1; k <= nWindows; ++k) {
        const double tk = (k == nWindows) ? tEnd : t0 + (double)k * hOuter;
        int rc = batch_impl(p, solver, t, tk, num, y, g, tol, stats, threads, 1);
        if (rc != BODE_OK) return rc;
        ++steps;
        t = tk;
    }
    if (outerSteps) *outerSteps = steps;
    return BODE_OK;
}

/* ------------------------------------------------------------------ */
/* glibc 2.39 cbrt, restated (sysdeps/ieee754/dbl-64/s_cbrt.c). The    */
/* reference calls libm cbrt (rkc.cpp:177-190); the device EXACT      */
/* policy evaluates this same algorithm (arith.cuh glibc_cbrt).       */
/* ------------------------------------------------------------------ */
double orc_glibc_cbrt(double x) {
    static const double factor[5] = {1.0 / 1.5874010519681994748, 1.0 / 1.2599210498948731648,
                                     1.0, 1.2599210498948731648, 1.5874010519681994748};
    int xe;
    const double xm = frexp(fabs(x), &xe);
    if (xe == 0 && fpclassify(x) <= FP_ZERO) return x + x;
    const double u =
        (0.354895765043919860 +
         ((1.50819193781584896 +
           ((-2.11499494167371287 +
             ((2.44693122563534430 +
               ((-1.83469277483613086 + (0.784932344976639262 - 0.145263899385486377 * xm) * xm) *
                xm)) *
              xm)) *
            xm)) *
          xm));
    const double t2 = u * u * u;
    const double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * factor[2 + xe % 3];
    return ldexp(x > 0.0 ? ym : -ym, xe / 3);
}

/* ------------------------------------------------------------------ */
/* glibc 2.39 pow, x86-64 FMA variant (__pow_fma, selected by ifunc on */
/* FMA/AVX2 hosts), restated from its instruction sequence: the ARM    */
/* optimized-routines algorithm (sysdeps/ieee754/dbl-64/e_pow.c) with  */
/* GCC's contractions. Tables (__pow_log_data, __exp_data) are read    */
/* from the libm loaded in this process, located by signature. The    */
/* reference calls pow in rkck::adjustStep (rkck.cpp:105, :109).       */
/* ------------------------------------------------------------------ */
#include <link.h>

typedef struct {
    const double* log_head; /* ln2hi, ln2lo, A[0..6], then tab[128][4] */
    const double* exp_head; /* invln2N, shift, negln2hiN, negln2loN, C2..C5 */
    const uint64_t* exp_tab; /* tab[256] */
} orc_powtab_t;

static orc_powtab_t g_powtab;
static int g_powtab_state = 0; /* 0 unknown, 1 found, -1 absent */

static const unsigned char* memfind(const unsigned char* h, size_t n, const void* pat, size_t m) {
    for (size_t i = 0; i + m <= n; i += 8)
        if (memcmp(h + i, pat, m) == 0) return h + i;
    return NULL;
}

static int phdr_cb(struct dl_phdr_info* info, size_t size, void* data) {
    (void)size;
    if (!info->dlpi_name || !strstr(info->dlpi_name, "libm.so")) return 0;
    orc_powtab_t* t = (orc_powtab_t*)data;
    const double log_sig[3] = {0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45, -0.5};
    const double exp_sig[2] = {0x1.71547652b82fep+7, 0x1.8p52};
    const uint64_t tab_sig[4] = {0x0ull, 0x3ff0000000000000ull, 0x3c9b3b4f1a88bf6eull,
                                 0x3feff63da9fb3335ull};
    for (int j = 0; j < info->dlpi_phnum; ++j) {
        const ElfW(Phdr)* ph = &info->dlpi_phdr[j];
        if (ph->p_type != PT_LOAD || !(ph->p_flags & PF_R) || (ph->p_flags & PF_X)) continue;
        const unsigned char* base = (const unsigned char*)(info->dlpi_addr + ph->p_vaddr);
        size_t n = ph->p_memsz & ~(size_t)7;
        base = (const unsigned char*)(((uintptr_t)base + 7) & ~(uintptr_t)7);
        if (!t->log_head) t->log_head = (const double*)memfind(base, n, log_sig, sizeof log_sig);
        if (!t->exp_head) t->exp_head = (const double*)memfind(base, n, exp_sig, sizeof exp_sig);
        if (!t->exp_tab) t->exp_tab = (const uint64_t*)memfind(base, n, tab_sig, sizeof tab_sig);
    }
    return 1;
}

int orc_glibc_pow_tables(const double** log_head, const double** exp_head,
                         const uint64_t** exp_tab) {
    if (g_powtab_state == 0) {
        memset(&g_powtab, 0, sizeof g_powtab);
        dl_iterate_phdr(phdr_cb, &g_powtab);
        g_powtab_state = (g_powtab.log_head && g_powtab.exp_head && g_powtab.exp_tab) ? 1 : -1;
    }
    if (g_powtab_state != 1) return 0;
    *log_head = g_powtab.log_head;
    *exp_head = g_powtab.exp_head;
    *exp_tab = g_powtab.exp_tab;
    return 1;
}

static inline uint64_t asu64(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double asf64(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

/* Main path only (x positive normal, 2^-65 <= |y| < 2^64, |y log x| < 512);
 * everything else returns libm pow itself (the reference's own value). */
double orc_glibc_pow(double x, double y) {
    const double *L, *E;
    const uint64_t* ET;
    const uint64_t ix = asu64(x), iy = asu64(y);
    const uint32_t topx = (uint32_t)(ix >> 52), topy = (uint32_t)(iy >> 52);
    if (!orc_glibc_pow_tables(&L, &E, &ET) || topx - 1u >= 0x7feu ||
        (topy & 0x7ffu) - 0x3beu > 0x7fu)
        return pow(x, y);
    /* log_inline */
    const uint64_t tmp = ix - 0x3fe6955500000000ull;
    const int i = (int)((tmp >> 45) & 0x7f);
    const int k = (int)((int64_t)tmp >> 52);
    const double z = asf64(ix - (tmp & 0xfff0000000000000ull));
    const double kd = (double)k;
    const double* T = L + 9 + 4 * i; /* invc, pad, logc, logctail */
    const double* A = L + 2;
    const double t1 = fma(kd, L[0], T[2]);
    const double lo1 = fma(kd, L[1], T[3]);
    const double r = fma(z, T[0], -1.0);
    const double ar = r * A[0];
    const double p12 = fma(r, A[2], A[1]);
    const double p34 = fma(r, A[4], A[3]);
    const double t2 = r + t1;
    const double lo2 = (t1 - t2) + r;
    const double ar2 = r * ar;
    const double ar3 = r * ar2;
    const double lo3 = fma(ar, r, -ar2);
    const double hi = t2 + ar2;
    const double p56 = fma(r, A[6], A[5]);
    const double lo4 = (t2 - hi) + ar2;
    const double q = fma(p56, ar2, p34);
    const double pp = fma(ar2, q, p12);
    double lo = ((lo1 + lo2) + lo3) + lo4;
    lo = fma(ar3, pp, lo);
    const double ly = hi + lo;
    const double ltail = (hi - ly) + lo;
    /* y * log(x) as ehi + elo */
    const double ehi = y * ly;
    const double elo = fma(y, ltail, fma(ly, y, -ehi));
    /* exp_inline */
    const uint32_t abstop = (uint32_t)(asu64(ehi) >> 52) & 0x7ffu;
    if (abstop - 0x3c9u > 0x3eu) {
        if (abstop - 0x3c9u >= 0x80000000u) return 1.0 + ehi; /* tiny: avoid spurious underflow */
        return pow(x, y);
    }
    double kk = fma(ehi, E[0], E[1]);
    const uint64_t ki = asu64(kk);
    kk = kk - E[1];
    double rr = fma(kk, E[2], ehi);
    rr = fma(kk, E[3], rr);
    rr = elo + rr;
    const uint64_t idx = 2 * (ki & 0x7f);
    const uint64_t top = ki << 45;
    const double tail = asf64(ET[idx]);
    const uint64_t sbits = ET[idx + 1] + top;
    double a = fma(rr, E[5], E[4]);
    const double b = rr + tail;
    const double r2 = rr * rr;
    const double c = fma(rr, E[7], E[6]);
    a = fma(a, r2, b);
    const double t = fma(c, r2 * r2, a);
    const double scale = asf64(sbits);
    return fma(scale, t, scale);
}
