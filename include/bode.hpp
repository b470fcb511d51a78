// bode.hpp -- C++20 drop-in for the reference's batch API, header-only over the
// C ABI (bode.h). Code written against batchode's headers
// (proj/include/batchode/{errors,ode_problem,batch,batch_driver,problems}.hpp)
// switches by replacing `batchode::` with `bode::` and linking libbode.so:
//
//   types          ToleranceSettings, IntegrationStats (camelCase fields,
//                  recordAcceptedStep, merge), SolverChoice, StepRecord, StepObserver,
//                  OdeProblem, BatchStates (at, gatherState, scatterState,
//                  gatherParams, validate), BatchResult, OuterLoopResult
//   batch helpers  pack, unpack, fillParams                     (batch.hpp:46-57)
//   entry points   integrateBatch(...), outerLoop(...)          (batch_driver.hpp:22-43)
//                  rkck::driver, rkck::integrateFixed, rkc::driver,
//                  rkc::integrateFixed (one system)       (rkck.hpp:73-83, rkc.hpp:116-128)
//   problems       pleiades(), heatEquation(n), expDecay(), harmonic(),
//                  loadPleiadesInitialConditions, fnv1aFileChecksum,
//                  pleiadesEnergy, pleiadesMomentum, heatSpectralRadius,
//                  heatInitialCondition, splitmix64At, unitSymmetricAt,
//                  perturbInitialConditions                     (problems.hpp:19-63)
//   errors         InvalidShape, InvalidInterval, InvalidStageCount,
//                  ConfigError, IoError                         (errors.hpp:8-30)
//
// The one difference inherent to a GPU drop-in: the right-hand side of an
// OdeProblem is a compiled device functor named by `kind` (a built-in problem,
// or one registered through include/bode_problem.cuh), not a host
// std::function -- there is no CPU fallback to run a host lambda on. Code that
// builds an OdeProblem from a lambda instead takes the matching device problem
// (e.g. problems::zero(dim) for the reference tests' zero RHS). `workers` is
// the number of shards (GPUs, or several shards per GPU); results are bitwise
// independent of it, as in the reference (batch_driver.hpp:16-21).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <exception>
#include <fstream>
#include <functional>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "bode.h"

namespace bode {

// ---- errors (errors.hpp:8-30) ----
struct InvalidShape : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct InvalidInterval : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct InvalidStageCount : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// A device-side failure (no CUDA device, CUDA runtime error, no kernel compiled
// for the problem): has no counterpart in the CPU reference.
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

// ---- ode_problem.hpp ----
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

struct IntegrationStats {  // ode_problem.hpp:57-81
    long stepsAccepted = 0;
    long stepsRejected = 0;
    long rhsEvals = 0;
    long specRadEvals = 0;
    double hMinSeen = std::numeric_limits<double>::infinity();
    double hMaxSeen = 0.0;
    bool underflow = false;
    long stagesTotal = 0;  // extension: sum of StepRecord.stages (ode_problem.hpp:90)

    void recordAcceptedStep(double h) {
        ++stepsAccepted;
        hMinSeen = std::min(hMinSeen, h);
        hMaxSeen = std::max(hMaxSeen, h);
    }
    void merge(const IntegrationStats& o) {
        stepsAccepted += o.stepsAccepted;
        stepsRejected += o.stepsRejected;
        rhsEvals += o.rhsEvals;
        specRadEvals += o.specRadEvals;
        stagesTotal += o.stagesTotal;
        hMinSeen = std::min(hMinSeen, o.hMinSeen);
        hMaxSeen = std::max(hMaxSeen, o.hMaxSeen);
        underflow = underflow || o.underflow;
    }
    static IntegrationStats from(const bode_stats_t& s) {
        IntegrationStats r;
        r.stepsAccepted = long(s.steps_accepted);
        r.stepsRejected = long(s.steps_rejected);
        r.rhsEvals = long(s.rhs_evals);
        r.specRadEvals = long(s.spec_rad_evals);
        r.stagesTotal = long(s.stages_total);
        r.hMinSeen = s.h_min_seen;
        r.hMaxSeen = s.h_max_seen;
        r.underflow = s.underflow != 0;
        return r;
    }
};

struct StepRecord {  // ode_problem.hpp:86-93
    double t;
    double h;
    int stages;
    double err;
    bool accepted;
};
// ode_problem.hpp:93: the per-attempt hook of the single-system drivers below
// (recorded on the device by bode_trace_steps and replayed in order).
using StepObserver = std::function<void(const StepRecord&)>;

// ode_problem.hpp:23-28 with the right-hand side named by a device problem kind.
struct OdeProblem {
    int dim = 0;
    int paramDim = 0;
    int kind = -1;  // BODE_PROBLEM_* or a registered kind; -1: no right-hand side
    bode_problem_t c() const { return {kind, dim, paramDim, 0}; }
};

// ---- batch.hpp ----
struct BatchStates {  // batch.hpp:15-45, values[i + numSystems*j]
    int numSystems = 0;
    int dim = 0;
    int paramDim = 0;
    std::vector<double> values;
    std::vector<double> params;

    double& at(int system, int var) {
        return values[std::size_t(system) + std::size_t(numSystems) * std::size_t(var)];
    }
    double at(int system, int var) const {
        return values[std::size_t(system) + std::size_t(numSystems) * std::size_t(var)];
    }
    void gatherState(int system, std::span<double> out) const {
        for (int j = 0; j < dim; ++j) out[j] = at(system, j);
    }
    void scatterState(int system, std::span<const double> in) {
        for (int j = 0; j < dim; ++j) at(system, j) = in[j];
    }
    void gatherParams(int system, std::span<double> out) const {
        for (int j = 0; j < paramDim; ++j)
            out[j] = params[std::size_t(system) + std::size_t(numSystems) * std::size_t(j)];
    }
    void validate() const {  // batch.cpp:8-22
        if (numSystems < 1 || dim < 1)
            throw InvalidShape("BatchStates: numSystems and dim must be positive");
        if (paramDim < 0) throw InvalidShape("BatchStates: negative paramDim");
        const std::size_t nv = std::size_t(numSystems) * std::size_t(dim);
        const std::size_t np = std::size_t(numSystems) * std::size_t(paramDim);
        if (values.size() != nv)
            throw InvalidShape("BatchStates: values length " + std::to_string(values.size()) +
                               " != numSystems*dim = " + std::to_string(nv));
        if (params.size() != np)
            throw InvalidShape("BatchStates: params length " + std::to_string(params.size()) +
                               " != numSystems*paramDim = " + std::to_string(np));
    }
};

// Interleaves per-system vectors into the SoA layout (batch.hpp:46-52).
inline BatchStates pack(const std::vector<std::vector<double>>& states,
                        const std::vector<std::vector<double>>& params = {}) {
    if (states.empty()) throw InvalidShape("pack: no systems");
    const std::size_t n = states.size(), d = states.front().size();
    if (d == 0) throw InvalidShape("pack: zero-dimensional state");
    for (const auto& s : states)
        if (s.size() != d) throw InvalidShape("pack: ragged state vectors");
    if (!params.empty() && params.size() != n)
        throw InvalidShape("pack: params count differs from state count");
    const std::size_t pd = params.empty() ? 0 : params.front().size();
    for (const auto& q : params)
        if (q.size() != pd) throw InvalidShape("pack: ragged parameter vectors");
    BatchStates b;
    b.numSystems = int(n);
    b.dim = int(d);
    b.paramDim = int(pd);
    b.values.resize(n * d);
    b.params.resize(n * pd);
    for (std::size_t j = 0; j < d; ++j)
        for (std::size_t i = 0; i < n; ++i) b.values[j * n + i] = states[i][j];
    for (std::size_t j = 0; j < pd; ++j)
        for (std::size_t i = 0; i < n; ++i) b.params[j * n + i] = params[i][j];
    return b;
}

// Inverse of pack for the state array (batch.hpp:54).
inline std::vector<std::vector<double>> unpack(const BatchStates& batch) {
    batch.validate();
    std::vector<std::vector<double>> out(std::size_t(batch.numSystems),
                                         std::vector<double>(std::size_t(batch.dim)));
    for (int i = 0; i < batch.numSystems; ++i) batch.gatherState(i, out[std::size_t(i)]);
    return out;
}

// The same parameter vector for every system (batch.hpp:56-57).
inline void fillParams(BatchStates& batch, std::span<const double> g) {
    batch.paramDim = int(g.size());
    batch.params.assign(std::size_t(batch.numSystems) * g.size(), 0.0);
    for (std::size_t j = 0; j < g.size(); ++j)
        std::fill_n(batch.params.begin() + std::ptrdiff_t(j * std::size_t(batch.numSystems)),
                    batch.numSystems, g[j]);
}

// ---- batch_driver.hpp ----
struct BatchResult {
    BatchStates states;
    std::vector<IntegrationStats> stats;  // one entry per system
};

using OuterStepSink = std::function<void(double t, BatchStates snapshot)>;

struct OuterLoopResult {
    BatchStates states;
    std::vector<IntegrationStats> stats;  // per system, summed over windows
    int outerSteps = 0;
};

// ---- problems.hpp ----
namespace problems {
inline constexpr int kPleiadesDim = 28;
inline constexpr std::uint64_t kPleiadesIcChecksum = 0x5583feb418028048ull;

// A built-in or registered device problem (bode_problem_init).
inline OdeProblem fromKind(int kind, int dim = 0) {
    bode_problem_t p{};
    check(bode_problem_init(&p, kind, dim));
    OdeProblem o;
    o.kind = p.kind;
    o.dim = p.dim;
    o.paramDim = p.param_dim;
    return o;
}
inline OdeProblem pleiades() { return fromKind(BODE_PROBLEM_PLEIADES); }
inline OdeProblem heatEquation(int interiorPoints) {
    if (interiorPoints < 2) throw InvalidShape("heatEquation: need at least two interior points");
    return fromKind(BODE_PROBLEM_HEAT, interiorPoints);
}
inline OdeProblem expDecay() { return fromKind(BODE_PROBLEM_EXPDECAY); }
inline OdeProblem harmonic() { return fromKind(BODE_PROBLEM_HARMONIC); }
// The reference tests' calibration right-hand sides, as device problems:
// y' = 0 (test_batch.cpp:80-89), y' = 1, y' = y^2, y' = sin(t) y, y_i' = g_i y_i.
inline OdeProblem zero(int dim) { return fromKind(BODE_PROBLEM_ZERO, dim); }
inline OdeProblem constant(int dim) { return fromKind(BODE_PROBLEM_CONST, dim); }
inline OdeProblem riccati() { return fromKind(BODE_PROBLEM_RICCATI); }
inline OdeProblem sinTimesY() { return fromKind(BODE_PROBLEM_SINT); }
inline OdeProblem diagonal(int dim) { return fromKind(BODE_PROBLEM_DIAG, dim); }

inline std::uint64_t splitmix64At(std::uint64_t seed, std::uint64_t k) {
    return bode_splitmix64_at(seed, k);
}
inline double unitSymmetricAt(std::uint64_t seed, std::uint64_t k) {
    return bode_unit_symmetric_at(seed, k);
}

// 28 whitespace-separated values (problems.cpp:39-53); IoError otherwise.
inline std::array<double, kPleiadesDim> loadPleiadesInitialConditions(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open Pleiades initial-condition file: " + path);
    std::array<double, kPleiadesDim> ic{};
    for (int i = 0; i < kPleiadesDim; ++i)
        if (!(in >> ic[std::size_t(i)]))
            throw IoError("Pleiades initial-condition file ends early or is non-numeric at line " +
                          std::to_string(i + 1) + ": " + path);
    double more;
    if (in >> more) throw IoError("Pleiades initial-condition file has more than 28 values: " + path);
    return ic;
}
// FNV-1a 64 over the file's bytes (problems.cpp:55-66).
inline std::uint64_t fnv1aFileChecksum(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open file for checksum: " + path);
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (int c = in.get(); c != std::char_traits<char>::eof(); c = in.get())
        h = (h ^ std::uint64_t(static_cast<unsigned char>(c))) * 0x100000001b3ull;
    return h;
}
inline std::vector<double> pleiadesInitialConditions() {
    std::vector<double> v(kPleiadesDim);
    bode_pleiades_ic(v.data());
    return v;
}
// Total energy and momentum of a Pleiades state (problems.cpp:68-92), the
// reference's drift oracles; masses m_i = i + 1.
inline double pleiadesEnergy(std::span<const double> w) {
    double kin = 0.0, pot = 0.0;
    for (int i = 0; i < 7; ++i)
        kin += 0.5 * double(i + 1) * (w[14 + i] * w[14 + i] + w[21 + i] * w[21 + i]);
    for (int i = 0; i < 7; ++i)
        for (int j = i + 1; j < 7; ++j) {
            const double dx = w[i] - w[j], dy = w[7 + i] - w[7 + j];
            pot -= double(i + 1) * double(j + 1) / std::sqrt(dx * dx + dy * dy);
        }
    return kin + pot;
}
inline std::array<double, 2> pleiadesMomentum(std::span<const double> w) {
    std::array<double, 2> p{0.0, 0.0};
    for (int i = 0; i < 7; ++i) {
        p[0] += double(i + 1) * w[14 + i];
        p[1] += double(i + 1) * w[21 + i];
    }
    return p;
}
// (4/dx^2) sin^2(n pi / (2(n+1))) (problems.cpp:117-122).
inline double heatSpectralRadius(int interiorPoints) {
    const double n = double(interiorPoints), dx = 1.0 / (n + 1.0);
    const double s = std::sin(n * 3.14159265358979323846 / (2.0 * (n + 1.0)));
    return 4.0 / (dx * dx) * s * s;
}
inline std::vector<double> heatInitialCondition(int interiorPoints) {
    std::vector<double> v(std::size_t(std::max(interiorPoints, 0)));
    bode_heat_initial_condition(interiorPoints, v.data());
    return v;
}
inline BatchStates perturbInitialConditions(std::span<const double> base, double magnitude,
                                            std::uint64_t seed, int count) {
    if (base.empty()) throw InvalidShape("perturbInitialConditions: empty base state");
    BatchStates b;
    b.numSystems = count;
    b.dim = int(base.size());
    b.values.resize(std::size_t(count > 0 ? count : 0) * base.size());
    check(bode_perturb_initial_conditions(base.data(), b.dim, magnitude, seed, count,
                                          b.values.data()));
    return b;
}
}  // namespace problems

namespace detail {
// batch_driver.cpp:42-50, in that order (the interval is checked first by the caller)
inline void checkCall(const OdeProblem& problem, const BatchStates& batch,
                      const ToleranceSettings& tol, int workers) {
    batch.validate();
    tol.validate();
    if (batch.dim != problem.dim)
        throw InvalidShape("integrateBatch: batch dim does not match problem dim");
    if (batch.paramDim != problem.paramDim)
        throw InvalidShape("integrateBatch: batch paramDim does not match problem");
    if (workers < 1) throw InvalidShape("integrateBatch: workers must be positive");
    if (problem.kind < 0) throw InvalidShape("integrateBatch: problem has no rhs");
}
inline std::vector<bode_stats_t> emptyStats(int n) {
    bode_stats_t s{};
    s.h_min_seen = std::numeric_limits<double>::infinity();
    return std::vector<bode_stats_t>(std::size_t(n), s);
}
inline std::vector<IntegrationStats> convert(const std::vector<bode_stats_t>& c) {
    std::vector<IntegrationStats> v(c.size());
    for (std::size_t i = 0; i < c.size(); ++i) v[i] = IntegrationStats::from(c[i]);
    return v;
}
}  // namespace detail

// batchode::integrateBatch (batch_driver.hpp:22-24). Validation order follows
// batch_driver.cpp:42-50: interval, shapes, tolerances, workers.
inline BatchResult integrateBatch(const OdeProblem& problem, const BatchStates& batch, double t,
                                  double tNext, SolverChoice solver,
                                  const ToleranceSettings& tol, int workers = 1,
                                  Arith arith = Arith::Exact) {
    if (!(tNext > t)) throw InvalidInterval("integrateBatch: tNext must exceed t");
    detail::checkCall(problem, batch, tol, workers);
    BatchResult r{batch, {}};
    auto st = detail::emptyStats(batch.numSystems);
    const bode_tol_t ct = tol.c();
    const bode_problem_t cp = problem.c();
    check(bode_int_driver(&cp, int(solver), int(arith), t, tNext, batch.numSystems,
                          r.states.params.empty() ? nullptr : r.states.params.data(),
                          r.states.values.data(), &ct, st.data(), workers));
    r.stats = detail::convert(st);
    return r;
}

// batchode::outerLoop (batch_driver.hpp:40-43): y stays on the device between
// windows; each snapshot is an independent copy handed to the sink in window
// order while later windows compute (batch_driver.hpp:26-28).
inline OuterLoopResult outerLoop(const OdeProblem& problem, const BatchStates& initial,
                                 double t0, double tEnd, double hOuter, SolverChoice solver,
                                 const ToleranceSettings& tol, int workers = 1,
                                 const OuterStepSink& sink = {}, Arith arith = Arith::Exact) {
    if (!(tEnd > t0)) throw InvalidInterval("outerLoop: tEnd must exceed t0");
    if (!(hOuter > 0.0)) throw InvalidInterval("outerLoop: hOuter must be positive");
    detail::checkCall(problem, initial, tol, workers);
    OuterLoopResult r{initial, {}, 0};
    auto st = detail::emptyStats(initial.numSystems);
    const bode_tol_t ct = tol.c();
    const bode_problem_t cp = problem.c();
    struct Ctx {
        const OuterStepSink* sink;
        const BatchStates* shape;
        std::exception_ptr error;
    } ctx{&sink, &initial, nullptr};
    bode_sink_fn fn = nullptr;
    if (sink)
        fn = [](double t, const double* y, int64_t num, int32_t dim, void* user) {
            auto* c = static_cast<Ctx*>(user);
            if (c->error) return;  // a previous sink threw: skip the rest
            try {
                BatchStates snap;
                snap.numSystems = c->shape->numSystems;
                snap.dim = c->shape->dim;
                snap.paramDim = c->shape->paramDim;
                snap.params = c->shape->params;
                snap.values.assign(y, y + num * dim);
                (*c->sink)(t, std::move(snap));
            } catch (...) {
                c->error = std::current_exception();
            }
        };
    int32_t steps = 0;
    check(bode_outer_loop(&cp, int(solver), int(arith), t0, tEnd, hOuter, initial.numSystems,
                          r.states.params.empty() ? nullptr : r.states.params.data(),
                          r.states.values.data(), &ct, st.data(), workers, fn, &ctx, &steps));
    if (ctx.error) std::rethrow_exception(ctx.error);
    r.stats = detail::convert(st);
    r.outerSteps = steps;
    return r;
}

namespace detail {
// One system (y, g) as a one-column batch through the C ABI.
inline IntegrationStats driveOne(const OdeProblem& problem, SolverChoice solver, double t,
                                 double tEnd, std::span<double> y, std::span<const double> g,
                                 const ToleranceSettings& tol, Arith arith) {
    if (!(tEnd > t))
        throw InvalidInterval(solver == SolverChoice::RKCK ? "rkck::driver: tEnd must exceed t"
                                                           : "rkc::driver: tEnd must exceed t");
    if (y.size() != std::size_t(problem.dim) || g.size() != std::size_t(problem.paramDim))
        throw InvalidShape("driver: state/parameter length does not match the problem");
    tol.validate();
    std::vector<bode_stats_t> st(1);
    const bode_tol_t ct = tol.c();
    const bode_problem_t cp = problem.c();
    check(bode_int_driver(&cp, int(solver), int(arith), t, tEnd, 1, g.empty() ? nullptr : g.data(),
                          y.data(), &ct, st.data(), 1));
    return convert(st)[0];
}
// driveOne with a StepObserver: the window runs once on the device with every
// attempt recorded (bode_trace_steps), then the records replay in order.
inline IntegrationStats driveObserved(const OdeProblem& problem, SolverChoice solver, double t,
                                      double tEnd, std::span<double> y,
                                      std::span<const double> g, const ToleranceSettings& tol,
                                      const StepObserver& observer, Arith arith) {
    if (!(tEnd > t))
        throw InvalidInterval(solver == SolverChoice::RKCK ? "rkck::driver: tEnd must exceed t"
                                                           : "rkc::driver: tEnd must exceed t");
    if (y.size() != std::size_t(problem.dim) || g.size() != std::size_t(problem.paramDim))
        throw InvalidShape("driver: state/parameter length does not match the problem");
    tol.validate();
    const bode_tol_t ct = tol.c();
    const bode_problem_t cp = problem.c();
    std::vector<bode_stats_t> st(1);
    std::vector<bode_step_record_t> rec(1024);
    std::vector<double> y0(y.begin(), y.end());
    int64_t n = 0;
    for (;;) {  // grow the record buffer until every attempt fits (re-running from y0)
        std::copy(y0.begin(), y0.end(), y.begin());
        check(bode_trace_steps(&cp, int(solver), int(arith), t, tEnd,
                               g.empty() ? nullptr : g.data(), y.data(), &ct, st.data(),
                               rec.data(), int64_t(rec.size()), &n));
        if (n <= int64_t(rec.size())) break;
        rec.resize(std::size_t(n));
    }
    if (observer)
        for (int64_t i = 0; i < n; ++i)
            observer(StepRecord{rec[i].t, rec[i].h, rec[i].stages, rec[i].err, rec[i].accepted != 0});
    return convert(st)[0];
}
inline void fixedOne(const OdeProblem& problem, SolverChoice solver, double t0, double tEnd,
                     long numSteps, int stages, double kappa, std::span<double> y,
                     std::span<const double> g, Arith arith) {
    if (y.size() != std::size_t(problem.dim) || g.size() != std::size_t(problem.paramDim))
        throw InvalidShape("integrateFixed: state/parameter length does not match the problem");
    const bode_problem_t cp = problem.c();
    check(bode_integrate_fixed(&cp, int(solver), int(arith), t0, tEnd, numSteps, stages, kappa, 1,
                               g.empty() ? nullptr : g.data(), y.data()));
}
}  // namespace detail

// The single-system entry points of the reference's solver headers
// (rkck.hpp:73-83, rkc.hpp:116-128), run on the device as a one-system batch.
// Scratch is accepted for source compatibility (the device needs none). The
// StepObserver overloads record every attempt on the device and replay the
// records; the RKC Workspace (the controller state left after the window) is
// not exported, so wsOut must be null.
namespace rkck {
struct Scratch {};  // rkck.hpp:22-31: per-thread buffers on the CPU; nothing to hold here
inline IntegrationStats driver(const OdeProblem& problem, double t, double tEnd,
                               std::span<double> y, std::span<const double> g,
                               const ToleranceSettings& tol, Scratch&,
                               const StepObserver* observer = nullptr,
                               Arith arith = Arith::Exact) {
    if (observer == nullptr)
        return detail::driveOne(problem, SolverChoice::RKCK, t, tEnd, y, g, tol, arith);
    return detail::driveObserved(problem, SolverChoice::RKCK, t, tEnd, y, g, tol, *observer, arith);
}
inline IntegrationStats driver(const OdeProblem& problem, double t, double tEnd,
                               std::span<double> y, std::span<const double> g,
                               const ToleranceSettings& tol = {}, Arith arith = Arith::Exact) {
    return detail::driveOne(problem, SolverChoice::RKCK, t, tEnd, y, g, tol, arith);
}
// rkck::integrateFixed (rkck.cpp:168-181)
inline void integrateFixed(const OdeProblem& problem, double t0, double tEnd, long numSteps,
                           std::span<double> y, std::span<const double> g,
                           Arith arith = Arith::Exact) {
    detail::fixedOne(problem, SolverChoice::RKCK, t0, tEnd, numSteps, 0, 0.0, y, g, arith);
}
}  // namespace rkck

namespace rkc {
struct Scratch {};    // rkc.hpp:52-64: CPU buffers; nothing to hold here
struct Workspace {};  // rkc.hpp:39-50: the controller state is not exported from the device
inline IntegrationStats driver(const OdeProblem& problem, double t, double tEnd,
                               std::span<double> y, std::span<const double> g,
                               const ToleranceSettings& tol, Scratch&, Workspace* wsOut = nullptr,
                               const StepObserver* observer = nullptr,
                               Arith arith = Arith::Exact) {
    if (wsOut != nullptr)
        throw InvalidShape("rkc::driver: the device controller state (Workspace) is not exported");
    if (observer == nullptr)
        return detail::driveOne(problem, SolverChoice::RKC, t, tEnd, y, g, tol, arith);
    return detail::driveObserved(problem, SolverChoice::RKC, t, tEnd, y, g, tol, *observer, arith);
}
inline IntegrationStats driver(const OdeProblem& problem, double t, double tEnd,
                               std::span<double> y, std::span<const double> g,
                               const ToleranceSettings& tol = {}, Arith arith = Arith::Exact) {
    return detail::driveOne(problem, SolverChoice::RKC, t, tEnd, y, g, tol, arith);
}
// rkc::integrateFixed (rkc.cpp:290-306)
inline void integrateFixed(const OdeProblem& problem, double t0, double tEnd, long numSteps,
                           int stages, double kappa, std::span<double> y,
                           std::span<const double> g, Arith arith = Arith::Exact) {
    detail::fixedOne(problem, SolverChoice::RKC, t0, tEnd, numSteps, stages, kappa, y, g, arith);
}
}  // namespace rkc

}  // namespace bode
