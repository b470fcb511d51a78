/*
 * bode_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm for the hot path
 * (arxiv/paper_1611_02274, batchode C++ library under /root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker. The product
 * (paper_1611_02274_b200/, include/bode.h) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference itself, compiled from its own sources into oracle/_ref/ (see
 * oracle/Makefile, tests/test_oracle_vs_ref.py), and against the reference
 * test suite's known-answer values (tests/test_oracle_kats.py).
 *
 * Problem ids, tolerance and stats layouts are shared with include/bode.h so
 * the checker and the product exchange the same structs.
 */
#ifndef BODE_ORACLE_H
#define BODE_ORACLE_H

#include <stdint.h>

#include "../include/bode.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Per-attempt observer, mirrors batchode::StepRecord (ode_problem.hpp:87-93). */
typedef void (*orc_observer_fn)(double t, double h, int stages, double err,
                                int accepted, void* user);

/* ---- problems (problems.cpp) ---- */
uint64_t orc_splitmix64_at(uint64_t seed, uint64_t k);
double orc_unit_symmetric_at(uint64_t seed, uint64_t k);
int orc_perturb(const double* base, int dim, double magnitude, uint64_t seed,
                int count, double* out_soa);
/* Evaluates the right-hand side of problem p (dim/param_dim given by p). */
void orc_rhs(const bode_problem_t* p, double t, const double* y, const double* g,
             double* out);
double orc_heat_spectral_radius(int n);
void orc_heat_initial_condition(int n, double* u);
double orc_pleiades_energy(const double* w);
void orc_pleiades_momentum(const double* w, double out[2]);

/* ---- RKCK (rkck.cpp) ---- */
void orc_rkck_step(const bode_problem_t* p, double t, const double* y,
                   const double* g, const double* f0, double h, double* yNext,
                   double* yErr);
void orc_rkck_error_norm(int n, const double* y, const double* f0,
                         const double* yErr, double h, double eps, double tiny,
                         double* err, int* nanFlag);
void orc_rkck_adjust_step(double h, double err, int nanFlag, double hMin,
                          double hMax, const bode_tol_t* tol, int* accepted,
                          double* hNew);
int orc_rkck_driver(const bode_problem_t* p, double t, double tEnd, double* y,
                    const double* g, const bode_tol_t* tol, bode_stats_t* st,
                    orc_observer_fn obs, void* user);
void orc_rkck_integrate_fixed(const bode_problem_t* p, double t0, double tEnd,
                              long numSteps, double* y, const double* g);

/* ---- RKC (rkc.cpp) ---- */
void orc_chebyshev_eval(int degree, double x, double out[3]);
/* Arrays must hold stages+1 doubles each. */
int orc_rkc_coefficients(int stages, double kappa, double* omega0, double* omega1,
                         double* mu, double* nu, double* muTilde,
                         double* gammaTilde, double* b, double* a, double* c);
int orc_rkc_step(const bode_problem_t* p, double t, const double* y,
                 const double* g, const double* f0, double h, int stages,
                 double kappa, double* yNext);
double orc_rkc_error_norm(int n, const double* yOld, const double* yNew,
                          const double* fOld, const double* fNew, double h,
                          double absTol, double relTol);
void orc_rkc_stage_count(double h, double sigma, double relTol, double uround,
                         int* stages, double* hOut);
void orc_rkc_initial_step(const bode_problem_t* p, double t, const double* y,
                          const double* g, const double* f0, double sigma,
                          double hMax, double hMin, const bode_tol_t* tol,
                          double* hOut, double* errOut);
double orc_rkc_next_step_accepted(double err, double errOld, double h,
                                  double hOld, int firstAccepted, double hMin,
                                  double hMax);
double orc_rkc_next_step_rejected(double err, double h);
int orc_rkc_driver(const bode_problem_t* p, double t, double tEnd, double* y,
                   const double* g, const bode_tol_t* tol, bode_stats_t* st,
                   orc_observer_fn obs, void* user);
void orc_rkc_integrate_fixed(const bode_problem_t* p, double t0, double tEnd,
                             long numSteps, int stages, double kappa, double* y,
                             const double* g);

/* ---- spectral radius (spectral_radius.cpp) ---- */
int orc_power_method(const bode_problem_t* p, double t, const double* y,
                     const double* g, const double* f0, double hMax,
                     const double* vWarm, double* sigma, double* eigvec,
                     int* iterations, int* converged);

/* glibc pow (x86-64 FMA build) restated; tables read from the loaded libm */
double orc_glibc_pow(double x, double y);
int orc_glibc_pow_tables(const double** log_head, const double** exp_head, const uint64_t** exp_tab);

/* glibc cbrt restated (see bode_oracle.c) */
double orc_glibc_cbrt(double x);

/* ---- batch layer (batch_driver.cpp) ---- */
/* y_soa / g_soa use the reference layout values[i + num*j]. stats: num entries. */
int orc_integrate_batch(const bode_problem_t* p, int solver, double t,
                        double tNext, int64_t num, double* y_soa,
                        const double* g_soa, const bode_tol_t* tol,
                        bode_stats_t* stats, int threads);
int orc_outer_loop(const bode_problem_t* p, int solver, double t0, double tEnd,
                   double hOuter, int64_t num, double* y_soa,
                   const double* g_soa, const bode_tol_t* tol,
                   bode_stats_t* stats, int threads, int* outerSteps);

#ifdef __cplusplus
}
#endif

#endif
