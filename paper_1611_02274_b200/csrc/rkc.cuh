// rkc.cuh -- adaptive Runge-Kutta-Chebyshev integration (with the
// Jacobian-free power-method spectral radius) of one system per lane group.
//
// Follows proj/src/rkc.cpp: chebyshevEval (:10-27), coefficients (:29-69),
// step (:82-117), errorNorm (:119-129), stageCount (:131-144), initialStep
// (:146-171), nextStepAccepted/Rejected (:173-191), driver (:193-281) and
// proj/src/spectral_radius.cpp powerMethod (:17-85).
//
// Differences in *form* only (results are bitwise the reference's with R=xd):
//  * Stage coefficients are generated on the fly by running the Chebyshev
//    recurrence alongside the stages instead of caching per-s vectors. The
//    reference evaluates chebyshevEval(j, x) from scratch for each j with the
//    same loop, so the j-th iterate is the same double; omega1 needs T'_s and
//    T''_s, obtained by a scalar pre-pass of s iterations.
//  * The driver loop is a small state machine (TOP -> [SPECRAD] -> ATTEMPT,
//    reject -> SPECRAD -> REJECT_TAIL) so the power method, the initial step
//    and the stage recurrence each have one call site in the kernel. The
//    event order per system is exactly the reference's.
//  * Sums that the reference accumulates sequentially (error norm, 2-norms)
//    stay sequential in component order across the lane group (seq_sum).
#pragma once

#include "rkck.cuh"

namespace bode {

// Running Chebyshev triple (T_j, T'_j, T''_j) at x (rkc.cpp:18-25).
template <class R>
struct Cheb {
    R T, d, dd;
};
template <class R>
__device__ __forceinline__ Cheb<R> cheb_next(const Cheb<R>& m1, const Cheb<R>& m2, R x) {
    Cheb<R> r;
    r.T = R(2.0) * x * m1.T - m2.T;
    r.d = R(2.0) * m1.T + R(2.0) * x * m1.d - m2.d;
    r.dd = R(4.0) * m1.d + R(2.0) * x * m1.dd - m2.dd;
    return r;
}

// Power method (spectral_radius.cpp:17-85). Returns sigma (with the 1.2
// safety factor) and the number of iterations (= RHS evaluations); eig is the
// warm start on entry and v - y on exit.
template <class P, class R, int L>
__device__ __forceinline__ int power_method(const Group<L>& G, R t, const R (&y)[P::N / L],
                                            const R* g, const R (&f0)[P::N / L], R hMax,
                                            R (&eig)[P::N / L], R& sigmaOut) {
    constexpr int C = P::N / L;
    constexpr int kItMax = 50;
    const R kUround(2.22e-16);
    const R sqrtU = sqrt_(kUround);
    const R small = R(1.0) / hMax;
    R v[C], tmp[C];
#pragma unroll
    for (int c = 0; c < C; ++c) tmp[c] = y[c] * y[c];
    const R nrmY = sqrt_(seq_sum<R, L, C>(G, tmp, R(0.0)));
#pragma unroll
    for (int c = 0; c < C; ++c) tmp[c] = eig[c] * eig[c];
    const R nrmV = sqrt_(seq_sum<R, L, C>(G, tmp, R(0.0)));
    R dynrm;
    if (nrmY != R(0.0) && nrmV != R(0.0)) {
        dynrm = nrmY * sqrtU;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = y[c] + eig[c] * (dynrm / nrmV);
    } else if (nrmY != R(0.0)) {
        dynrm = nrmY * sqrtU;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = y[c] * (R(1.0) + sqrtU);
    } else if (nrmV != R(0.0)) {
        dynrm = kUround;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = eig[c] * (dynrm / nrmV);
    } else {
        dynrm = kUround;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = kUround;
    }
    R sigma(0.0);
    int iters = 0;
#pragma unroll 1
    for (int iter = 1; iter <= kItMax; ++iter) {
        R fv[C];
        P::template rhs<R, L>(G, t, v, g, fv);
        iters = iter;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const R d = fv[c] - f0[c];
            tmp[c] = d * d;
        }
        const R diffNrm = sqrt_(seq_sum<R, L, C>(G, tmp, R(0.0)));
        const R sigmaOld = sigma;
        sigma = diffNrm / dynrm;
        if (iter >= 2 && fabs_(sigma - sigmaOld) <= fmax_(sigma, small) * R(0.01)) break;
        if (diffNrm != R(0.0)) {
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = y[c] + (fv[c] - f0[c]) * (dynrm / diffNrm);
        } else {  // degenerate direction: flip one component about y
            const int ind = iter % P::N;
#pragma unroll
            for (int c = 0; c < C; ++c)
                if (G.lane * C + c == ind) v[c] = y[c] - (v[c] - y[c]);
        }
    }
    sigmaOut = R(1.2) * sigma;
#pragma unroll
    for (int c = 0; c < C; ++c) eig[c] = v[c] - y[c];
    return iters;
}

// One RKC stage j >= 2 (rkc.cpp:99-112): dst <- w_j from src = w_{j-1} and
// dst = w_{j-2} on entry (ignored when first, i.e. w_{j-2} = y).
template <class P, class R, int L>
__device__ __forceinline__ void rkc_stage(const Group<L>& G, R tj, const R (&y)[P::N / L],
                                          const R (&f0)[P::N / L], const R* g,
                                          const R (&src)[P::N / L], R (&dst)[P::N / L], R muj,
                                          R nuj, R mujh, R gjh, bool first) {
    constexpr int C = P::N / L;
    R f[C];
    P::template rhs<R, L>(G, tj, src, g, f);
    if (first) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            dst[c] = y[c] + muj * (src[c] - y[c]) + mujh * f[c] + gjh * f0[c];
    } else {
#pragma unroll
        for (int c = 0; c < C; ++c)
            dst[c] = y[c] + muj * (src[c] - y[c]) + nuj * (dst[c] - y[c]) + mujh * f[c] +
                     gjh * f0[c];
    }
}

enum RkcState { kTop = 0, kSrThenAttempt = 1, kAttempt = 2, kSrThenRejectTail = 3, kRejectTail = 4 };

// rkc::driver (rkc.cpp:193-281) for this lane group's system.
template <class P, class R, int L>
__device__ __forceinline__ void rkc_system(const Group<L>& G, double t_in, double tEnd_in,
                                           R (&y)[P::N / L], const R* g, const DevTol& tol,
                                           DevStats& st) {
    constexpr int C = P::N / L;
    stats_init(st);
    const R tEnd(tEnd_in);
    R t(t_in);
    const R uround(tol.uround), absTol(tol.abs_tol), relTol(tol.rel_tol), kappa(tol.kappa);
    const R hMax = fabs_(tEnd - t);
    // stageCount's mMax (rkc.cpp:132-133), a per-call constant
    long long mMax = llround(val(sqrt_(relTol / (R(10.0) * uround))));
    if (mMax < 2) mMax = 2;

    R wsErrOld(0.0), wsHOld(0.0), wsH(0.0), wsSpecRad(0.0);  // Workspace::reset
    long long numStep = 0;
    R f0[C], eig[C];
    P::template rhs<R, L>(G, t, y, g, f0);
    ++st.rhs_evals;
#pragma unroll
    for (int c = 0; c < C; ++c) eig[c] = f0[c];  // rkc.cpp:212

    int state = kTop;
    R hMin(0.0), hNewRej(0.0);
#pragma unroll 1
    for (;;) {
        if (state == kTop) {
            if (!(tEnd - t > uround * fabs_(tEnd))) break;
            hMin = R(10.0) * uround * fmax_(fabs_(t), hMax);
            if (R(1.1) * wsH >= fabs_(tEnd - t)) wsH = fabs_(tEnd - t);
            state = (numStep % 25 == 0) ? kSrThenAttempt : kAttempt;
        }
        if (state == kSrThenAttempt || state == kSrThenRejectTail) {
            R sig;
            const int it = power_method<P, R, L>(G, t, y, g, f0, hMax, eig, sig);
            wsSpecRad = sig;
            ++st.spec_rad_evals;
            st.rhs_evals += it;
            state = (state == kSrThenAttempt) ? kAttempt : kRejectTail;
        }
        if (state == kRejectTail) {
            if (hNewRej < hMin) {  // freeze at the last accepted state (rkc.cpp:260-263)
                st.underflow = 1;
                break;
            }
            wsH = hNewRej;
            state = kTop;
            continue;
        }
        // ---- state == kAttempt ----
        R wa[C], wb[C];
        if (wsH < uround) {  // initialStep (rkc.cpp:146-171), one RHS
            R h = hMax;
            if (wsSpecRad * h > R(1.0)) h = R(1.0) / wsSpecRad;
            h = fmax_(h, hMin);
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = y[c] + h * f0[c];
            P::template rhs<R, L>(G, t + h, wa, g, wb);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const R est = (wb[c] - f0[c]) / (absTol + relTol * fabs_(y[c]));
                wa[c] = est * est;
            }
            const R sum = seq_sum<R, L, C>(G, wa, R(0.0));
            const R err = h * sqrt_(sum / R(double(P::N)));
            if (R(0.1) * h < hMax * sqrt_(err))
                h = fmax_(R(0.1) * h / sqrt_(err), hMin);
            else
                h = hMax;
            ++st.rhs_evals;
            wsH = h;
        }
        const R sigma = isfinite_(wsSpecRad) ? wsSpecRad : R(0.0);
        // stageCount (rkc.cpp:131-144)
        long long s;
        {
            const R raw = sqrt_(R(1.54) * wsH * sigma + R(1.0));
            s = (raw < R(double(mMax))) ? 1 + (long long)val(raw) : mMax + 1;
            if (s > mMax) {
                s = mMax;
                wsH = (R(double(s)) * R(double(s)) - R(1.0)) / (R(1.54) * sigma);
            }
        }
        const R h = wsH;
        // coefficients (rkc.cpp:29-69): omega0, then omega1 = T'_s / T''_s
        const R omega0 = R(1.0) + kappa / (R(double(s)) * R(double(s)));
        R omega1;
        {
            Cheb<R> m2{R(1.0), R(0.0), R(0.0)}, m1{omega0, R(1.0), R(0.0)};
#pragma unroll 1
            for (long long j = 2; j <= s; ++j) {
                const Cheb<R> cur = cheb_next(m1, m2, omega0);
                m2 = m1;
                m1 = cur;
            }
            omega1 = m1.d / m1.dd;
        }
        // ---- rkc::step (rkc.cpp:82-117) ----
        const R b1 = R(1.0) / omega0;
        {
            const R mu1h = (b1 * omega1) * h;  // muTilde_1 * h
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = y[c] + mu1h * f0[c];
        }
        // Chebyshev state: Tm1 = T_{j-1}, Tm2 = T_{j-2}; bm1 = b_{j-1}, bm2 = b_{j-2}
        Cheb<R> Tm2{R(1.0), R(0.0), R(0.0)}, Tm1{omega0, R(1.0), R(0.0)};
        R bm1 = b1, bm2(0.0);
        const Cheb<R> T2 = cheb_next(Tm1, Tm2, omega0);
        const R b2 = T2.dd / (T2.d * T2.d);
        bm2 = b2;  // b_0 = b_2 (rkc.cpp:50), only reached through nu_2 (unused)
        // c_1 = c_2 / (4 omega0), c_2 interior unless s == 2 (then c_2 = c_s = 1)
        const R c2 = (s > 2) ? omega1 * T2.dd / T2.d : R(1.0);
        R cjm1 = c2 / (R(4.0) * omega0);  // c_{j-1} at j = 2
        R am1 = R(1.0) - b1 * Tm1.T;      // a_1
        bool inA = true;                   // current w_{j-1} lives in wa
#pragma unroll 1
        for (long long j = 2; j <= s; ++j) {
            const Cheb<R> Tj = (j == 2) ? T2 : cheb_next(Tm1, Tm2, omega0);
            const R bj = (j == 2) ? b2 : Tj.dd / (Tj.d * Tj.d);
            const R muj = R(2.0) * bj * omega0 / bm1;
            const R nuj = -bj / bm2;
            const R muTj = R(2.0) * bj * omega1 / bm1;
            const R gTj = -am1 * muTj;
            const R tj = t + cjm1 * h;
            if (inA)
                rkc_stage<P, R, L>(G, tj, y, f0, g, wa, wb, muj, nuj, muTj * h, gTj * h, j == 2);
            else
                rkc_stage<P, R, L>(G, tj, y, f0, g, wb, wa, muj, nuj, muTj * h, gTj * h, false);
            inA = !inA;
            // advance to j+1: c_j (interior for j < s), a_j, b's, T's
            cjm1 = (j < s) ? omega1 * Tj.dd / Tj.d : R(1.0);
            am1 = R(1.0) - bj * Tj.T;
            bm2 = bm1;
            bm1 = bj;
            Tm2 = Tm1;
            Tm1 = Tj;
        }
        if (!inA) {  // y_trial = w_s -> wa
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = wb[c];
        }
        st.rhs_evals += s - 1;
        st.stages_total += s;
        P::template rhs<R, L>(G, t + h, wa, g, wb);  // f_trial (rkc.cpp:247)
        ++st.rhs_evals;
        // errorNorm (rkc.cpp:119-129)
        R err;
        {
            R terms[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                R est = R(0.8) * (y[c] - wa[c]) + R(0.4) * h * (f0[c] + wb[c]);
                est = est / (absTol + relTol * fmax_(fabs_(y[c]), fabs_(wa[c])));
                terms[c] = est * est;
            }
            err = sqrt_(seq_sum<R, L, C>(G, terms, R(0.0)) / R(double(P::N)));
        }
        const bool accepted = err <= R(1.0);
        if (!accepted) {
            ++st.steps_rejected;
            hNewRej = isfinite_(err) ? R(0.8) * h / cbrt_(err) : R(tol.p1) * h;
            state = kSrThenRejectTail;
        } else {
            t += h;
            ++numStep;
            stats_accept(st, val(h));
            const bool firstAccepted = wsHOld < uround;
            // nextStepAccepted (rkc.cpp:173-187)
            R fac(10.0);
            if (firstAccepted) {
                const R t2 = cbrt_(err);
                if (R(0.8) < fac * t2) fac = R(0.8) / t2;
            } else {
                const R t1 = R(0.8) * h * cbrt_(wsErrOld);
                const R cb = cbrt_(err);
                const R t2 = wsHOld * cb * cb;
                if (t1 < fac * t2) fac = t1 / t2;
            }
            const R hNew = fmax_(hMin, fmin_(hMax, h * fmax_(R(0.1), fac)));
            wsErrOld = fmax_(err, uround);
            wsHOld = h;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                y[c] = wa[c];
                f0[c] = wb[c];  // FSAL swap (rkc.cpp:276)
            }
            wsH = hNew;
            state = kTop;
        }
    }
}

}  // namespace bode
