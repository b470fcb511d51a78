// rkck.cuh -- adaptive Runge-Kutta-Cash-Karp integration of one system per
// lane group, entirely on chip.
//
// Follows proj/src/rkck.cpp: tableau (:8-27), step (:34-78), errorNorm
// (:88-98), adjustStep (:100-113) and driver (:115-159). The step, its
// embedded error estimate, the scaled max-norm and the controller are fused:
// yErr is never materialised, it is folded into the norm component by
// component, and yNext is formed in place only once the step is accepted.
//
// Storage: y and f0 live in registers. The stage derivatives k2..k5 live in
// registers for small systems or in shared memory for large ones (KSMEM),
// one odd-length row per thread (conflict-free, immediate-offset addressing).
// k6 stays in the RHS output registers.
#pragma once

#include "dispatch.h"
#include "problems.cuh"

namespace bode {

__device__ __forceinline__ void stats_init(DevStats& s) {
    s.steps_accepted = s.steps_rejected = s.rhs_evals = s.spec_rad_evals = s.stages_total = 0;
    s.h_min_seen = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    s.h_max_seen = 0.0;
    s.underflow = 0;
    s.budget_exhausted = 0;
}

// IntegrationStats::recordAcceptedStep (ode_problem.hpp:66-70)
__device__ __forceinline__ void stats_accept(DevStats& s, double h) {
    ++s.steps_accepted;
    s.h_min_seen = fmin(s.h_min_seen, h);
    s.h_max_seen = fmax(s.h_max_seen, h);
}

// IntegrationStats::merge (ode_problem.hpp:72-80)
__device__ __forceinline__ void stats_merge(DevStats& a, const DevStats& b) {
    a.steps_accepted += b.steps_accepted;
    a.steps_rejected += b.steps_rejected;
    a.rhs_evals += b.rhs_evals;
    a.spec_rad_evals += b.spec_rad_evals;
    a.stages_total += b.stages_total;
    a.h_min_seen = fmin(a.h_min_seen, b.h_min_seen);
    a.h_max_seen = fmax(a.h_max_seen, b.h_max_seen);
    a.underflow = a.underflow || b.underflow;
    a.budget_exhausted = a.budget_exhausted || b.budget_exhausted;
}

// The opt-in per-window attempt budget (bode_set_attempt_budget; not in the
// reference, off by default). A register countdown: no stats loads on the
// serial controller path. When it runs out, the caller freezes the system at
// its last accepted state, as on underflow.
#ifndef BODE_ATTEMPT_BUDGET
#define BODE_ATTEMPT_BUDGET 1
#endif
// Kernels are compiled with and without it (the INSTR template mode: 0 plain,
// 1 budget, 2 budget and step trace; the host launches an instrumented
// instance only while a budget or a trace is requested), so the default path
// carries no budget code at all.
template <bool ON = true>
struct AttemptBudget {
    long long left;  // attempts still allowed (no budget: more than any window makes)
    __device__ __forceinline__ void init(const DevTol& tol) {
        left = tol.max_attempts > 0 ? tol.max_attempts : 0x7fffffffffffffffll;
    }
    // before an attempt: true (and the stats flag) if none is left, else charges one
    __device__ __forceinline__ bool spent(DevStats& st) {
        if (!BODE_ATTEMPT_BUDGET) return false;
        if (left <= 0) {
            st.budget_exhausted = 1;
            return true;
        }
        --left;
        return false;
    }
    // after an attempt of a system that is still live: charges it and reports
    // whether that was the last one allowed
    __device__ __forceinline__ bool spent_after(DevStats& st) {
        if (!BODE_ATTEMPT_BUDGET) return false;
        if (--left <= 0) {
            st.budget_exhausted = 1;
            return true;
        }
        return false;
    }
};
// StepObserver (ode_problem.hpp:85-94, invoked at rkck.cpp:142 and rkc.cpp:253):
// in the instrumented kernel instances only, the lead lane of a traced
// one-system launch appends (t, h, stages, err, accepted) for every attempt.
template <bool ON, class R>
__device__ __forceinline__ void trace_step(const DevTol& tol, bool lead, R t, R h, int stages,
                                           R err, bool accepted) {
    if constexpr (ON) {
        if (tol.trace != nullptr && lead) {
            const unsigned long long i = atomicAdd(tol.trace_count, 1ull);
            if (i < (unsigned long long)tol.trace_cap)
                tol.trace[i] = StepRec{val(t), val(h), val(err), stages, accepted ? 1 : 0};
        }
    }
}

template <>
struct AttemptBudget<false> {
    __device__ __forceinline__ void init(const DevTol&) {}
    __device__ __forceinline__ bool spent(DevStats&) { return false; }
    __device__ __forceinline__ bool spent_after(DevStats&) { return false; }
};

// Cash-Karp tableau (rkck.cpp:8-27), evaluated as the same double quotients.
namespace ck {
constexpr double a2 = 1.0 / 5.0, a3 = 3.0 / 10.0, a4 = 3.0 / 5.0, a5 = 1.0, a6 = 7.0 / 8.0;
constexpr double b21 = 1.0 / 5.0;
constexpr double b31 = 3.0 / 40.0, b32 = 9.0 / 40.0;
constexpr double b41 = 3.0 / 10.0, b42 = -9.0 / 10.0, b43 = 6.0 / 5.0;
constexpr double b51 = -11.0 / 54.0, b52 = 5.0 / 2.0, b53 = -70.0 / 27.0, b54 = 35.0 / 27.0;
constexpr double b61 = 1631.0 / 55296.0, b62 = 175.0 / 512.0, b63 = 575.0 / 13824.0,
                 b64 = 44275.0 / 110592.0, b65 = 253.0 / 4096.0;
constexpr double c1 = 37.0 / 378.0, c3 = 250.0 / 621.0, c4 = 125.0 / 594.0, c5 = 0.0,
                 c6 = 512.0 / 1771.0;
constexpr double s1 = 2825.0 / 27648.0, s3 = 18575.0 / 48384.0, s4 = 13525.0 / 55296.0,
                 s5 = 277.0 / 14336.0, s6 = 1.0 / 4.0;
// d = c - c* (rkck.cpp:68-72); both operands are exact double constants and
// the subtraction is a single IEEE rounding, folded at compile time.
constexpr double d1 = c1 - s1, d3 = c3 - s3, d4 = c4 - s4, d5 = c5 - s5, d6 = c6 - s6;
}  // namespace ck

// Shared-memory row length per thread for 4 stage slots of C doubles: rounded
// up to an odd number of doubles so the 64-bit accesses of a half-warp hit 16
// distinct bank pairs (conflict-free) while every address is base + immediate.
template <int C>
__host__ __device__ constexpr int kSmemStride() { return (4 * C) | 1; }

// Stage-derivative store for k2..k5 (slot 0..3).
template <class R, int C, bool SMEM>
struct KStore;

template <class R, int C>
struct KStore<R, C, false> {
    R k[4][C];
    __device__ __forceinline__ R get(int m, int c) const { return k[m][c]; }
    __device__ __forceinline__ void set(int m, int c, R v) { k[m][c] = v; }
};

template <class R, int C>
struct KStore<R, C, true> {
    double* base;  // dynamic shared memory: one row of kSmemStride<C>() doubles per thread
    __device__ __forceinline__ KStore() {
        extern __shared__ double bode_smem[];
        base = bode_smem + threadIdx.x * kSmemStride<C>();
    }
    __device__ __forceinline__ R get(int m, int c) const { return R(base[m * C + c]); }
    __device__ __forceinline__ void set(int m, int c, R v) { base[m * C + c] = val(v); }
};

// adjustStep (rkck.cpp:100-113)
template <class R>
__device__ __forceinline__ bool rkck_adjust(R h, R err, bool nanFlag, R hMin, R hMax,
                                            const DevTol& tol, R& hNew) {
    // one pow call site (it is large under EXACT: glibc's algorithm inline)
    // with the exponent of whichever branch needs it: the same bits as two
    const bool reject = err > R(1.0) || !isfinite_(err) || nanFlag;
    const bool bad = !isfinite_(err) || nanFlag;
    R pw(1.0);
    if ((reject && !bad) || (!reject && err > R(tol.errcon)))
        pw = pow_(err, R(reject ? tol.pshrnk : tol.pgrow), tol.powtab);  // FAST: ctrl_pow_fast
    if (reject) {
        hNew = bad ? R(tol.p1) * h : fmax_(R(tol.safety) * h * pw, R(tol.p1) * h);
        return false;
    }
    const R hn = (err > R(tol.errcon)) ? R(tol.safety) * h * pw : R(5.0) * h;
    hNew = fmax_(hMin, fmin_(hMax, hn));
    return true;
}

// One system (this lane's slice) from t to tEnd: rkck::driver (rkck.cpp:115-159).
// y is updated in place; returns the window's stats.
template <class P, class R, int L, bool KSMEM, int INSTR>
__device__ __forceinline__ void rkck_system(const Group<L>& G, double t_in, double tEnd_in,
                                            R (&y)[P::N / L], const R* g, const DevTol& tol,
                                            DevStats& st) {
    constexpr int C = P::N / L;
    using namespace ck;
    stats_init(st);
    const R tEnd(tEnd_in);
    R t(t_in);
    const R hMax = fabs_(tEnd - t);
    const R hMin(tol.h_min_floor);
    R h = R(0.5) * fabs_(tEnd - t);
    const R uround(tol.uround), eps(tol.eps), tiny(tol.tiny);

    R f0[C];
    KStore<R, C, KSMEM> K;
    bool haveF = false;
    AttemptBudget<(INSTR >= 1)> bud;
    bud.init(tol);

#pragma unroll 1
    while (tEnd - t > uround * fabs_(tEnd)) {
        if (bud.spent(st)) break;
        h = fmin_(tEnd - t, h);
        R arg[C], out[C];
        if (!haveF) {  // rejected retries reuse f(t, y) (rkck.cpp:133-137)
            P::template rhs<R, L>(G, t, y, g, f0);
            ++st.rhs_evals;
            haveF = true;
        }
        // ---- rkck::step (rkck.cpp:42-64): five stage evaluations ----
        // The newest stage derivative is the last term of every stage sum, so
        // it is read from the RHS output registers (`out`) rather than reloaded
        // -- the reference's summation order is unchanged. FAST folds h into
        // the weights (one FMA per term).
        const R hh = h;
        auto stage_arg = [&](int c, double w1, const double* wk, int nk, R newest, double wn) -> R {
            if constexpr (is_exact<R>::value) {
                R s = R(w1) * f0[c];
                for (int m = 0; m < nk; ++m) s = s + R(wk[m]) * K.get(m, c);
                s = s + R(wn) * newest;
                return y[c] + hh * s;
            } else {
                double s = fma(val(hh) * w1, val(f0[c]), val(y[c]));
                for (int m = 0; m < nk; ++m) s = fma(val(hh) * wk[m], val(K.get(m, c)), s);
                return R(fma(val(hh) * wn, val(newest), s));
            }
        };
        // stage 2: y + h*b21*f0
#pragma unroll
        for (int c = 0; c < C; ++c) arg[c] = y[c] + h * R(b21) * f0[c];
        P::template rhs<R, L>(G, t + R(a2) * h, arg, g, out);
        // stage 3
        {
            const double w[1] = {0.0};
#pragma unroll
            for (int c = 0; c < C; ++c) {
                arg[c] = stage_arg(c, b31, w, 0, out[c], b32);
                K.set(0, c, out[c]);
            }
        }
        P::template rhs<R, L>(G, t + R(a3) * h, arg, g, out);
        // stage 4
        {
            const double w[1] = {b42};
#pragma unroll
            for (int c = 0; c < C; ++c) {
                arg[c] = stage_arg(c, b41, w, 1, out[c], b43);
                K.set(1, c, out[c]);
            }
        }
        P::template rhs<R, L>(G, t + R(a4) * h, arg, g, out);
        // stage 5
        {
            const double w[2] = {b52, b53};
#pragma unroll
            for (int c = 0; c < C; ++c) {
                arg[c] = stage_arg(c, b51, w, 2, out[c], b54);
                K.set(2, c, out[c]);
            }
        }
        P::template rhs<R, L>(G, t + R(a5) * h, arg, g, out);
        // stage 6
        {
            const double w[3] = {b62, b63, b64};
#pragma unroll
            for (int c = 0; c < C; ++c) {
                arg[c] = stage_arg(c, b61, w, 3, out[c], b65);
                K.set(3, c, out[c]);
            }
        }
        P::template rhs<R, L>(G, t + R(a6) * h, arg, g, out);  // out = k6
        st.rhs_evals += 5;
        st.stages_total += 6;

        // ---- yErr folded into errorNorm (rkck.cpp:75-76, :88-98) ----
        R err(0.0);
        bool nanFlag = false;
        if constexpr (is_exact<R>::value) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const R yErr = h * (R(d1) * f0[c] + R(d3) * K.get(1, c) + R(d4) * K.get(2, c) +
                                    R(d5) * K.get(3, c) + R(d6) * out[c]);
                if (!isfinite_(yErr)) nanFlag = true;
                err = fmax_(err, fabs_(yErr / (fabs_(y[c]) + fabs_(h * f0[c]) + tiny)));
            }
            if constexpr (L > 1) {
                err = R(G.max_all(val(err)));
                nanFlag = G.any(nanFlag);
            }
            err = err / eps;
        } else {
            // FAST: argmax of |e|/d by cross-multiplication, one reciprocal; the
            // candidate yNext goes into arg (free now), in the same pass
            const double hv = val(h);
            const double hd1 = hv * d1, hd3 = hv * d3, hd4 = hv * d4, hd5 = hv * d5, hd6 = hv * d6;
            const double hc1 = hv * c1, hc3 = hv * c3, hc4 = hv * c4, hc6 = hv * c6;
            double ma = 0.0, mb = 1.0;
            int bad = 0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const double k3 = val(K.get(1, c)), k4 = val(K.get(2, c)), k6 = val(out[c]);
                const double e = fma(hd6, k6, fma(hd5, val(K.get(3, c)),
                                 fma(hd4, k4, fma(hd3, k3, hd1 * val(f0[c])))));
                arg[c] = R(fma(hc6, k6, fma(hc4, k4, fma(hc3, k3, fma(hc1, val(f0[c]), val(y[c]))))));
                bad |= (__double2hiint(e) & 0x7ff00000) == 0x7ff00000;
                const double d = fma(hv, fabs(val(f0[c])), fabs(val(y[c]))) + val(tiny);
                if (fabs(e) * mb > ma * d) { ma = fabs(e); mb = d; }
            }
            if constexpr (L > 1) {
#pragma unroll
                for (int o = L / 2; o > 0; o /= 2) {
                    const double oa = __shfl_xor_sync(G.mask, ma, o, L);
                    const double ob = __shfl_xor_sync(G.mask, mb, o, L);
                    if (oa * mb > ma * ob) { ma = oa; mb = ob; }
                }
                nanFlag = G.any(bad != 0);
            } else {
                nanFlag = bad != 0;
            }
            err = R(ma * rcp_fast(mb * val(eps)));
        }

        R hNew;
        const bool accepted = rkck_adjust(h, err, nanFlag, hMin, hMax, tol, hNew);
        trace_step<(INSTR == 2)>(tol, G.lane == 0, t, h, 6, err, accepted);
        if (accepted) {
            t += h;
            stats_accept(st, val(h));
            // yNext (rkck.cpp:74), written over y once the step is accepted
            if constexpr (is_exact<R>::value) {
#pragma unroll
                for (int c = 0; c < C; ++c)
                    y[c] = y[c] + h * (R(c1) * f0[c] + R(c3) * K.get(1, c) + R(c4) * K.get(2, c) +
                                       R(c6) * out[c]);
            } else {
#pragma unroll
                for (int c = 0; c < C; ++c) y[c] = arg[c];
            }
            haveF = false;
            h = hNew;
        } else {
            ++st.steps_rejected;
            if (hNew < R(tol.h_min_floor)) {  // freeze at the last accepted state
                st.underflow = 1;
                break;
            }
            h = hNew;
        }
    }
}

}  // namespace bode
