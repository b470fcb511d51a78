// bode.hpp -- C++ drop-in for the reference's batch API, header-only over the
// C ABI (bode.h). A translation unit using batchode's integrateBatch /
// outerLoop (proj/include/batchode/batch_driver.hpp:22-43) switches by
// replacing `batchode::` with `bode::` and linking libbode.so:
//
//   types          ToleranceSettings, IntegrationStats, SolverChoice, BatchStates,
//                  BatchResult, OuterLoopResult        (ode_problem.hpp, batch.hpp)
//   problems       pleiades(), heatEquation(n), expDecay(), harmonic(),
//                  perturbInitialConditions(...)        (problems.hpp:19-63)
//   entry points   integrateBatch(...), outerLoop(...)  (batch_driver.hpp:22-43)
//   errors         InvalidShape, InvalidInterval, InvalidStageCount (errors.hpp)
//
// One difference is inherent to a GPU drop-in: OdeProblem names a compiled
// device right-hand side (Problem kind + shape) instead of holding a host
// std::function, and `workers` becomes the number of GPUs. Results are
// bitwise independent of it, as in the reference (batch_driver.hpp:16-21).
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "bode.h"

namespace bode {

struct InvalidShape : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct InvalidInterval : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct InvalidStageCount : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == BODE_OK) return;
    const std::string msg = bode_last_error();
    switch (rc) {
        case BODE_E_INVALID_INTERVAL: throw InvalidInterval(msg);
        case BODE_E_INVALID_SHAPE: throw InvalidShape(msg);
        case BODE_E_INVALID_STAGE_COUNT: throw InvalidStageCount(msg);
        default: throw DeviceError(msg);
    }
}

enum class SolverChoice { RKCK = BODE_SOLVER_RKCK, RKC = BODE_SOLVER_RKC };
enum class Arith { Exact = BODE_ARITH_EXACT, Fast = BODE_ARITH_FAST };

struct ToleranceSettings {  // ode_problem.hpp:32-54
    double eps = 1.0e-10, absTol = 1.0e-10, relTol = 1.0e-6, uround = 2.22e-16,
           tiny = 1.0e-30, safety = 0.9, p1 = 0.1, errcon = 1.89e-4, pgrow = -0.2,
           pshrnk = -0.25, hMinFloor = 1.0e-20, kappa = 2.0 / 13.0;
    bode_tol_t c() const {
        return {eps, absTol, relTol, uround, tiny, safety, p1, errcon, pgrow, pshrnk, hMinFloor,
                kappa};
    }
    void validate() const {
        const bode_tol_t t = c();
        check(bode_tol_validate(&t));
    }
};

using IntegrationStats = bode_stats_t;  // ode_problem.hpp:57-81 (+ stages_total)

struct OdeProblem {  // ode_problem.hpp:23-28, RHS selected by kind
    bode_problem_t p{};
    int dim() const { return p.dim; }
    int paramDim() const { return p.param_dim; }
};

struct BatchStates {  // batch.hpp:15-45, values[i + numSystems*j]
    int numSystems = 0, dim = 0, paramDim = 0;
    std::vector<double> values, params;
    double& at(int system, int var) { return values[std::size_t(system) + std::size_t(numSystems) * var]; }
    double at(int system, int var) const { return values[std::size_t(system) + std::size_t(numSystems) * var]; }
    void validate() const {  // batch.cpp:8-22
        if (numSystems < 1 || dim < 1) throw InvalidShape("BatchStates: numSystems and dim must be positive");
        if (paramDim < 0) throw InvalidShape("BatchStates: negative paramDim");
        if (values.size() != std::size_t(numSystems) * dim)
            throw InvalidShape("BatchStates: values length != numSystems*dim");
        if (params.size() != std::size_t(numSystems) * paramDim)
            throw InvalidShape("BatchStates: params length != numSystems*paramDim");
    }
};

struct BatchResult {
    BatchStates states;
    std::vector<IntegrationStats> stats;
};

struct OuterLoopResult {
    BatchStates states;
    std::vector<IntegrationStats> stats;
    int outerSteps = 0;
};

using OuterStepSink = std::function<void(double t, BatchStates snapshot)>;

namespace problems {
inline OdeProblem make(int kind, int dim = 0) {
    OdeProblem p;
    check(bode_problem_init(&p.p, kind, dim));
    return p;
}
inline OdeProblem pleiades() { return make(BODE_PROBLEM_PLEIADES); }
inline OdeProblem heatEquation(int interiorPoints) { return make(BODE_PROBLEM_HEAT, interiorPoints); }
inline OdeProblem expDecay() { return make(BODE_PROBLEM_EXPDECAY); }
inline OdeProblem harmonic() { return make(BODE_PROBLEM_HARMONIC); }
inline std::vector<double> pleiadesInitialConditions() {
    std::vector<double> v(28);
    bode_pleiades_ic(v.data());
    return v;
}
inline std::vector<double> heatInitialCondition(int n) {
    std::vector<double> v(n);
    bode_heat_initial_condition(n, v.data());
    return v;
}
inline BatchStates perturbInitialConditions(const std::vector<double>& base, double magnitude,
                                            std::uint64_t seed, int count) {
    BatchStates b;
    b.numSystems = count;
    b.dim = int(base.size());
    b.values.resize(std::size_t(count > 0 ? count : 0) * base.size());
    check(bode_perturb_initial_conditions(base.data(), b.dim, magnitude, seed, count, b.values.data()));
    return b;
}
}  // namespace problems

namespace detail {
inline void checkBatch(const OdeProblem& problem, const BatchStates& batch) {
    batch.validate();
    if (batch.dim != problem.dim()) throw InvalidShape("integrateBatch: batch dim does not match problem dim");
    if (batch.paramDim != problem.paramDim())
        throw InvalidShape("integrateBatch: batch paramDim does not match problem");
}
inline std::vector<IntegrationStats> emptyStats(int n) {
    IntegrationStats s{};
    s.h_min_seen = std::numeric_limits<double>::infinity();
    return std::vector<IntegrationStats>(std::size_t(n), s);
}
}  // namespace detail

// batchode::integrateBatch (batch_driver.hpp:22-24); gpus plays the role of workers.
inline BatchResult integrateBatch(const OdeProblem& problem, const BatchStates& batch, double t,
                                  double tNext, SolverChoice solver,
                                  const ToleranceSettings& tol, int gpus = 1,
                                  Arith arith = Arith::Exact) {
    if (!(tNext > t)) throw InvalidInterval("integrateBatch: tNext must exceed t");
    detail::checkBatch(problem, batch);
    tol.validate();
    BatchResult r{batch, detail::emptyStats(batch.numSystems)};
    const bode_tol_t ct = tol.c();
    check(bode_int_driver(&problem.p, int(solver), int(arith), t, tNext, batch.numSystems,
                          r.states.params.empty() ? nullptr : r.states.params.data(),
                          r.states.values.data(), &ct, r.stats.data(), gpus));
    return r;
}

// batchode::outerLoop (batch_driver.hpp:40-43): y stays on the device between windows.
inline OuterLoopResult outerLoop(const OdeProblem& problem, const BatchStates& initial,
                                 double t0, double tEnd, double hOuter, SolverChoice solver,
                                 const ToleranceSettings& tol, int gpus = 1,
                                 const OuterStepSink& sink = {}, Arith arith = Arith::Exact) {
    if (!(tEnd > t0)) throw InvalidInterval("outerLoop: tEnd must exceed t0");
    if (!(hOuter > 0.0)) throw InvalidInterval("outerLoop: hOuter must be positive");
    detail::checkBatch(problem, initial);
    tol.validate();
    OuterLoopResult r{initial, detail::emptyStats(initial.numSystems), 0};
    const bode_tol_t ct = tol.c();
    struct Ctx {
        const OuterStepSink* sink;
        BatchStates* states;
    } ctx{&sink, &r.states};
    bode_sink_fn fn = nullptr;
    if (sink)
        fn = [](double t, const double* y, int64_t num, int32_t dim, void* user) {
            auto* c = static_cast<Ctx*>(user);
            BatchStates snap = *c->states;
            snap.values.assign(y, y + num * dim);
            (*c->sink)(t, std::move(snap));
        };
    int32_t steps = 0;
    check(bode_outer_loop(&problem.p, int(solver), int(arith), t0, tEnd, hOuter,
                          initial.numSystems,
                          r.states.params.empty() ? nullptr : r.states.params.data(),
                          r.states.values.data(), &ct, r.stats.data(), gpus, fn, &ctx, &steps));
    r.outerSteps = steps;
    return r;
}

}  // namespace bode
