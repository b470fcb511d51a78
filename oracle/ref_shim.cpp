// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C entry points over the UNMODIFIED reference library, which oracle/Makefile
// compiles from /root/reference/proj/src into oracle/_ref/libbatchode_ref.so.
// Used to pin the C restatement (bode_oracle.c) bit for bit and as the
// reference CPU arm of bench.py (`--impl reference`). Nothing here is part
// of the product.
#include <cmath>
#include <cstring>
#include <vector>

#include "batchode/batch.hpp"
#include "batchode/batch_driver.hpp"
#include "batchode/problems.hpp"
#include "batchode/rkc.hpp"
#include "batchode/rkck.hpp"
#include "batchode/spectral_radius.hpp"
#ifdef BODE_REF_HAVE_BENCH
#include "batchode/bench.hpp"
#endif

#include "../include/bode.h"

using namespace batchode;

namespace {

OdeProblem makeProblem(const bode_problem_t* p) {
    switch (p->kind) {
        case BODE_PROBLEM_PLEIADES: return problems::pleiades();
        case BODE_PROBLEM_HEAT: return problems::heatEquation(p->dim);
        case BODE_PROBLEM_EXPDECAY: return problems::expDecay();
        case BODE_PROBLEM_HARMONIC: return problems::harmonic();
        default: break;
    }
    OdeProblem q;
    q.dim = p->dim;
    q.paramDim = p->param_dim;
    switch (p->kind) {
        case BODE_PROBLEM_ZERO:
            q.rhs = [](double, std::span<const double>, std::span<const double>,
                       std::span<double> out) {
                for (auto& x : out) x = 0.0;
            };
            break;
        case BODE_PROBLEM_RICCATI:
            q.rhs = [](double, std::span<const double> y, std::span<const double>,
                       std::span<double> out) { out[0] = y[0] * y[0]; };
            break;
        case BODE_PROBLEM_DIAG:
            q.rhs = [](double, std::span<const double> y, std::span<const double> g,
                       std::span<double> out) {
                for (std::size_t i = 0; i < y.size(); ++i) out[i] = g[i] * y[i];
            };
            break;
        case BODE_PROBLEM_CONST:
            q.rhs = [](double, std::span<const double>, std::span<const double>,
                       std::span<double> out) {
                for (auto& x : out) x = 1.0;
            };
            break;
        case BODE_PROBLEM_SINT:
            q.rhs = [](double t, std::span<const double> y, std::span<const double>,
                       std::span<double> out) { out[0] = std::sin(t) * y[0]; };
            break;
        case BODE_PROBLEM_BRUSSELATOR:
            // Not a reference problem: the host form of the device Brusselator
            // (paper_1611_02274_b200/csrc/problems_ext.cu), written as a user of
            // the reference would write an OdeProblem, so the reference drivers
            // integrate it. y = (u_1, v_1, ..., u_n, v_n), g = (A, B, alpha),
            // boundary values (A, B/A), stencil (1, -2, 1)/dx^2, dx = 1/(n+1).
            q.rhs = [](double, std::span<const double> y, std::span<const double> g,
                       std::span<double> out) {
                const int n = static_cast<int>(y.size()) / 2;
                const double A = g[0], B = g[1], alpha = g[2];
                const double dx = 1.0 / (n + 1);
                const double c = alpha / (dx * dx);
                const double ub = A, vb = B / A;
                for (int i = 0; i < n; ++i) {
                    const double u = y[2 * i], v = y[2 * i + 1];
                    const double uL = i > 0 ? y[2 * i - 2] : ub;
                    const double vL = i > 0 ? y[2 * i - 1] : vb;
                    const double uR = i < n - 1 ? y[2 * i + 2] : ub;
                    const double vR = i < n - 1 ? y[2 * i + 3] : vb;
                    const double uuv = u * u * v;
                    out[2 * i] = A + uuv - (B + 1.0) * u + c * (uL - 2.0 * u + uR);
                    out[2 * i + 1] = B * u - uuv + c * (vL - 2.0 * v + vR);
                }
            };
            break;
        default: break;
    }
    return q;
}

ToleranceSettings toTol(const bode_tol_t* t) {
    ToleranceSettings s;
    s.eps = t->eps;
    s.absTol = t->abs_tol;
    s.relTol = t->rel_tol;
    s.uround = t->uround;
    s.tiny = t->tiny;
    s.safety = t->safety;
    s.p1 = t->p1;
    s.errcon = t->errcon;
    s.pgrow = t->pgrow;
    s.pshrnk = t->pshrnk;
    s.hMinFloor = t->h_min_floor;
    s.kappa = t->kappa;
    return s;
}

void toStats(const IntegrationStats& s, bode_stats_t* o, long stages) {
    o->steps_accepted = s.stepsAccepted;
    o->steps_rejected = s.stepsRejected;
    o->rhs_evals = s.rhsEvals;
    o->spec_rad_evals = s.specRadEvals;
    o->stages_total = stages;
    o->h_min_seen = s.hMinSeen;
    o->h_max_seen = s.hMaxSeen;
    o->underflow = s.underflow ? 1 : 0;
    o->budget_exhausted = 0;
}

BatchStates toBatch(const bode_problem_t* p, int64_t num, const double* y, const double* g) {
    BatchStates b;
    b.numSystems = static_cast<int>(num);
    b.dim = p->dim;
    b.paramDim = p->param_dim;
    b.values.assign(y, y + num * p->dim);
    if (p->param_dim > 0) b.params.assign(g, g + num * p->param_dim);
    return b;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return BODE_OK;
    } catch (const InvalidInterval&) {
        return BODE_E_INVALID_INTERVAL;
    } catch (const InvalidShape&) {
        return BODE_E_INVALID_SHAPE;
    } catch (const InvalidStageCount&) {
        return BODE_E_INVALID_STAGE_COUNT;
    } catch (...) {
        return BODE_E_CUDA;
    }
}

}  // namespace

extern "C" {

// batchode::outerLoop with the reference's own std::thread worker pool.
// stats (nullable) are the reference's merged per-system stats; stages_total
// is not tracked by the reference batch layer and is reported as -1.
int ref_outer_loop(const bode_problem_t* p, int solver, double t0, double tEnd,
                   double hOuter, int64_t num, double* y, const double* g,
                   const bode_tol_t* tol, bode_stats_t* stats, int workers,
                   int* outerSteps) {
    return guarded([&] {
        const BatchStates b = toBatch(p, num, y, g);
        const OuterLoopResult r =
            outerLoop(makeProblem(p), b, t0, tEnd, hOuter,
                      solver == BODE_SOLVER_RKCK ? SolverChoice::RKCK : SolverChoice::RKC,
                      toTol(tol), workers, {});
        std::memcpy(y, r.states.values.data(), sizeof(double) * r.states.values.size());
        if (stats)
            for (int64_t i = 0; i < num; ++i) toStats(r.stats[i], &stats[i], -1);
        if (outerSteps) *outerSteps = r.outerSteps;
    });
}

int ref_integrate_batch(const bode_problem_t* p, int solver, double t, double tNext,
                        int64_t num, double* y, const double* g, const bode_tol_t* tol,
                        bode_stats_t* stats, int workers) {
    return guarded([&] {
        const BatchStates b = toBatch(p, num, y, g);
        const BatchResult r = integrateBatch(
            makeProblem(p), b, t, tNext,
            solver == BODE_SOLVER_RKCK ? SolverChoice::RKCK : SolverChoice::RKC,
            toTol(tol), workers);
        std::memcpy(y, r.states.values.data(), sizeof(double) * r.states.values.size());
        if (stats)
            for (int64_t i = 0; i < num; ++i) toStats(r.stats[i], &stats[i], -1);
    });
}

// batchode::outerLoop on an OdeProblem whose rhs is a C function pointer:
// the oracle for problems registered from user libraries, whose host form
// the library exports (e.g. examples/user_problem.cu).
typedef void (*ref_rhs_fn)(double t, const double* y, const double* g, double* out);
int ref_outer_loop_fn(ref_rhs_fn rhs, int dim, int param_dim, int solver, double t0,
                      double tEnd, double hOuter, int64_t num, double* y, const double* g,
                      const bode_tol_t* tol, bode_stats_t* stats, int workers,
                      int* outerSteps) {
    return guarded([&] {
        bode_problem_t p{BODE_PROBLEM_USER_BASE, dim, param_dim, 0};
        const BatchStates b = toBatch(&p, num, y, g);
        OdeProblem q;
        q.dim = dim;
        q.paramDim = param_dim;
        q.rhs = [rhs](double t, std::span<const double> yy, std::span<const double> gg,
                      std::span<double> out) { rhs(t, yy.data(), gg.data(), out.data()); };
        const OuterLoopResult r =
            outerLoop(q, b, t0, tEnd, hOuter,
                      solver == BODE_SOLVER_RKCK ? SolverChoice::RKCK : SolverChoice::RKC,
                      toTol(tol), workers, {});
        std::memcpy(y, r.states.values.data(), sizeof(double) * r.states.values.size());
        if (stats)
            for (int64_t i = 0; i < num; ++i) toStats(r.stats[i], &stats[i], -1);
        if (outerSteps) *outerSteps = r.outerSteps;
    });
}

// Single-system drivers with an observer that sums StepRecord.stages.
int ref_driver(const bode_problem_t* p, int solver, double t, double tEnd, double* y,
               const double* g, const bode_tol_t* tol, bode_stats_t* st) {
    return guarded([&] {
        long stages = 0;
        StepObserver obs = [&](const StepRecord& r) { stages += r.stages; };
        std::span<double> ys(y, p->dim);
        std::span<const double> gs(g, g ? p->param_dim : 0);
        IntegrationStats s;
        if (solver == BODE_SOLVER_RKCK) {
            rkck::Scratch sc;
            s = rkck::driver(makeProblem(p), t, tEnd, ys, gs, toTol(tol), sc, &obs);
        } else {
            rkc::Scratch sc;
            s = rkc::driver(makeProblem(p), t, tEnd, ys, gs, toTol(tol), sc, nullptr, &obs);
        }
        toStats(s, st, stages);
    });
}

uint64_t ref_splitmix64_at(uint64_t seed, uint64_t k) { return problems::splitmix64At(seed, k); }

int ref_perturb(const double* base, int dim, double magnitude, uint64_t seed, int count,
                double* out) {
    return guarded([&] {
        const BatchStates b = problems::perturbInitialConditions(
            std::span<const double>(base, dim), magnitude, seed, count);
        std::memcpy(out, b.values.data(), sizeof(double) * b.values.size());
    });
}

int ref_load_pleiades_ic(const char* path, double* out) {
    return guarded([&] {
        const auto ic = problems::loadPleiadesInitialConditions(path);
        std::memcpy(out, ic.data(), sizeof(double) * ic.size());
    });
}

uint64_t ref_fnv1a(const char* path) { return problems::fnv1aFileChecksum(path); }

void ref_rhs(const bode_problem_t* p, double t, const double* y, const double* g,
             double* out) {
    makeProblem(p).rhs(t, std::span<const double>(y, p->dim),
                       std::span<const double>(g, g ? p->param_dim : 0),
                       std::span<double>(out, p->dim));
}

void ref_rkck_step(const bode_problem_t* p, double t, const double* y, const double* g,
                   const double* f0, double h, double* yNext, double* yErr) {
    const int n = p->dim;
    const auto r = rkck::step(makeProblem(p), t, std::span<const double>(y, n),
                              std::span<const double>(g, g ? p->param_dim : 0),
                              std::span<const double>(f0, n), h);
    std::memcpy(yNext, r.yNext.data(), sizeof(double) * n);
    std::memcpy(yErr, r.yErr.data(), sizeof(double) * n);
}

void ref_rkck_adjust_step(double h, double err, int nanFlag, double hMin, double hMax,
                          const bode_tol_t* tol, int* accepted, double* hNew) {
    const auto a = rkck::adjustStep(h, err, nanFlag != 0, hMin, hMax, toTol(tol));
    *accepted = a.accepted ? 1 : 0;
    *hNew = a.hNew;
}

int ref_rkc_coefficients(int stages, double kappa, double* omega0, double* omega1,
                         double* mu, double* nu, double* muTilde, double* gammaTilde,
                         double* b, double* a, double* c) {
    return guarded([&] {
        const rkc::Coefficients cf = rkc::coefficients(stages, kappa);
        *omega0 = cf.omega0;
        *omega1 = cf.omega1;
        for (int j = 0; j <= stages; ++j) {
            mu[j] = cf.mu[j];
            nu[j] = cf.nu[j];
            muTilde[j] = cf.muTilde[j];
            gammaTilde[j] = cf.gammaTilde[j];
            b[j] = cf.b[j];
            a[j] = cf.a[j];
            c[j] = cf.c[j];
        }
    });
}

int ref_rkc_step(const bode_problem_t* p, double t, const double* y, const double* g,
                 const double* f0, double h, int stages, double kappa, double* yNext) {
    return guarded([&] {
        const int n = p->dim;
        rkc::Scratch sc;
        rkc::step(makeProblem(p), t, std::span<const double>(y, n),
                  std::span<const double>(g, g ? p->param_dim : 0),
                  std::span<const double>(f0, n), h, rkc::coefficients(stages, kappa),
                  std::span<double>(yNext, n), sc);
    });
}

void ref_rkc_stage_count(double h, double sigma, double relTol, double uround, int* s,
                         double* hOut) {
    const auto sel = rkc::stageCount(h, sigma, relTol, uround);
    *s = sel.stages;
    *hOut = sel.h;
}

double ref_rkc_next_step_accepted(double err, double errOld, double h, double hOld,
                                  int first, double hMin, double hMax) {
    return rkc::nextStepAccepted(err, errOld, h, hOld, first != 0, hMin, hMax);
}

double ref_rkc_next_step_rejected(double err, double h) {
    return rkc::nextStepRejected(err, h);
}

int ref_power_method(const bode_problem_t* p, double t, const double* y, const double* g,
                     const double* f0, double hMax, const double* vWarm, double* sigma,
                     double* eig, int* iterations, int* converged) {
    return guarded([&] {
        const int n = p->dim;
        const auto r = specrad::powerMethod(
            makeProblem(p), t, std::span<const double>(y, n),
            std::span<const double>(g, g ? p->param_dim : 0),
            std::span<const double>(f0, n), hMax, std::span<const double>(vWarm, n));
        *sigma = r.sigma;
        std::memcpy(eig, r.eigenvector.data(), sizeof(double) * n);
        *iterations = r.iterations;
        *converged = r.converged ? 1 : 0;
    });
}

#ifdef BODE_REF_HAVE_BENCH
// batchode::bench::run (bench.cpp:382-397): the reference's odebench minus
// its CLI11 front end, for comparing report files with bode's odebench.
int ref_bench_run(const char* problem, const char* solver, const char* mode, int numSystems,
                  double t0, double tEnd, double hOuter, double eps, double absTol,
                  double relTol, int workers, uint64_t seed, double perturb,
                  const char* output, const char* summary, const char* icPath,
                  int heatPoints) {
    try {
        bench::RunConfig cfg;
        cfg.problem = bench::parseProblem(problem);
        cfg.solver = bench::parseSolver(solver);
        cfg.mode = bench::parseMode(mode);
        cfg.numSystems = numSystems;
        cfg.t0 = t0;
        cfg.tEnd = tEnd;
        cfg.hOuter = hOuter;
        cfg.eps = eps;
        cfg.absTol = absTol;
        cfg.relTol = relTol;
        cfg.workers = workers;
        cfg.seed = seed;
        cfg.perturbMagnitude = perturb;
        cfg.outputPath = output ? output : "";
        cfg.summaryPath = summary ? summary : "";
        cfg.pleiadesIcPath = icPath ? icPath : "";
        cfg.heatPoints = heatPoints;
        return bench::run(cfg);
    } catch (...) {
        return 2;
    }
}
#endif

}  // extern "C"
