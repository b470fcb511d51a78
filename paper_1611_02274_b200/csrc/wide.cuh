// wide.cuh -- one system per thread block, for systems whose dimension is a
// run-time value: heatEquation(n) for any n >= 2 (problems.cpp:94-115), up to
// the reference's own dim-1e6 smoke size (test_rkc.cpp:491-512).
//
// The lane-group kernels (rkck.cuh, rkc.cuh) hold a system in registers and
// are compiled per dimension; this path keeps the state-length vectors of a
// system in shared memory when they fit (8 n doubles <= kWideSmemMax) and in
// a per-block global scratch otherwise, and the block's threads stride over
// the components. Scalars (t, h, the controller state, the stats) are kept
// redundantly by every thread: each computes the same IEEE operations on the
// same operands, so the control flow is block-uniform without broadcasts.
// Values that come out of a reduction are broadcast through shared memory.
//
// Follows, with the same expression shapes as the lane-group kernels (so the
// EXACT policy is bitwise the reference's):
//   rkck::step / errorNorm / adjustStep / driver   rkck.cpp:34-78, :88-159
//   rkc::step / errorNorm / initialStep / driver   rkc.cpp:82-129, :146-171, :193-281
//   specrad::powerMethod                           spectral_radius.cpp:17-85
// Sequential sums (rkc.cpp:122-127, spectral_radius.cpp:11-13) run in index
// order on one thread under EXACT; FAST reduces them as a tree.
#pragma once

#include "rkc.cuh"

namespace bode {

// kWideVecs, kWideMaxBlock, kWideSmemMax, wide_block: dispatch.h

// Heat equation with n interior points, n a run-time value (problems.cpp:94-115).
struct HeatWide {
    static constexpr int kind = 1, P = 0;
    // out <- f(t, u) over the block; u must be complete (caller syncs)
    template <class R>
    __device__ __forceinline__ static void rhs(int n, double invDx2, R, const double* u,
                                               double* out) {
        const R inv(invDx2);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            if (i == 0)
                out[i] = val((R(-2.0) * R(u[0]) + R(u[1])) * inv);
            else if (i == n - 1)
                out[i] = val((R(u[n - 2]) - R(2.0) * R(u[n - 1])) * inv);
            else
                out[i] = val((R(u[i - 1]) - R(2.0) * R(u[i]) + R(u[i + 1])) * inv);
        }
    }
    // the problem's constant 1/dx^2 with dx = 1/(n+1), as the reference forms it
    __device__ __forceinline__ static double inv_dx2(int n) {
        const double dx = __ddiv_rn(1.0, double(n + 1));
        return __ddiv_rn(1.0, __dmul_rn(dx, dx));
    }
};

// Block-wide reductions. `red` is a shared array of >= 33 doubles.
__device__ __forceinline__ double block_max(double* red, double v) {
#pragma unroll
    for (int o = 16; o > 0; o /= 2) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o /= 2) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (threadIdx.x == 0) red[32] = w;
    }
    __syncthreads();
    return red[32];
}
__device__ __forceinline__ bool block_any(bool b) { return __syncthreads_or(b ? 1 : 0) != 0; }

// Sum of terms[0..n) (written by the block before the call). EXACT: the
// reference's `s += term` in index order, on thread 0; FAST: a tree.
template <class R>
__device__ __forceinline__ R block_sum(double* red, const double* terms, int n) {
    if constexpr (is_exact<R>::value) {
        __syncthreads();
        if (threadIdx.x == 0) {
            R s(0.0);
            int i = 0;
            for (; i + 8 <= n; i += 8) {  // loads issued ahead of the dependent adds
                double v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = terms[i + k];
#pragma unroll
                for (int k = 0; k < 8; ++k) s = s + R(v[k]);
            }
            for (; i < n; ++i) s = s + R(terms[i]);
            red[32] = val(s);
        }
        __syncthreads();
        return R(red[32]);
    } else {
        double p = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) p += terms[i];
#pragma unroll
        for (int o = 16; o > 0; o /= 2) p += __shfl_xor_sync(0xffffffffu, p, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
        __syncthreads();
        if (threadIdx.x < 32) {
            double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o /= 2) w += __shfl_xor_sync(0xffffffffu, w, o);
            if (threadIdx.x == 0) red[32] = w;
        }
        __syncthreads();
        return R(red[32]);
    }
}

// The system's vectors (each n doubles) and the problem's run-time shape.
struct WideVecs {
    double *y, *f0, *a, *b, *c, *d, *e, *f;
    int n;
    double inv;  // problem constant (heat: 1/dx^2)
    double* red;
};

// f(t, u) into out between block barriers (the RHS reads neighbours of u,
// and the next writer of u must not overtake a reader).
template <class Prob, class R>
__device__ __forceinline__ void wide_rhs(const WideVecs& V, R t, const double* u, double* out) {
    __syncthreads();
    Prob::template rhs<R>(V.n, V.inv, t, u, out);
    __syncthreads();
}

// rkck::step's five stage evaluations (rkck.cpp:42-64): k2..k6 in V.a..V.e
// from y and f0 = f(t, y), the stage argument in V.f.
template <class Prob, class R>
__device__ __forceinline__ void rkck_wide_stages(const WideVecs& V, R t, R h, const double* y,
                                                 const double* f0) {
    using namespace ck;
    const int n = V.n;
    double *k2 = V.a, *k3 = V.b, *k4 = V.c, *k5 = V.d, *k6 = V.e, *yt = V.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        yt[i] = val(R(y[i]) + h * R(b21) * R(f0[i]));
    wide_rhs<Prob, R>(V, t + R(a2) * h, yt, k2);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        yt[i] = val(R(y[i]) + h * (R(b31) * R(f0[i]) + R(b32) * R(k2[i])));
    wide_rhs<Prob, R>(V, t + R(a3) * h, yt, k3);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        yt[i] = val(R(y[i]) + h * (R(b41) * R(f0[i]) + R(b42) * R(k2[i]) + R(b43) * R(k3[i])));
    wide_rhs<Prob, R>(V, t + R(a4) * h, yt, k4);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        yt[i] = val(R(y[i]) + h * (R(b51) * R(f0[i]) + R(b52) * R(k2[i]) + R(b53) * R(k3[i]) +
                                   R(b54) * R(k4[i])));
    wide_rhs<Prob, R>(V, t + R(a5) * h, yt, k5);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        yt[i] = val(R(y[i]) + h * (R(b61) * R(f0[i]) + R(b62) * R(k2[i]) + R(b63) * R(k3[i]) +
                                   R(b64) * R(k4[i]) + R(b65) * R(k5[i])));
    wide_rhs<Prob, R>(V, t + R(a6) * h, yt, k6);
}

// yNext (rkck.cpp:74) over y in place
template <class R>
__device__ __forceinline__ void rkck_wide_update(const WideVecs& V, R h, double* y,
                                                 const double* f0) {
    using namespace ck;
    for (int i = threadIdx.x; i < V.n; i += blockDim.x)
        y[i] = val(R(y[i]) + h * (R(c1) * R(f0[i]) + R(c3) * R(V.b[i]) + R(c4) * R(V.c[i]) +
                                  R(c6) * R(V.e[i])));
}

// rkck::driver (rkck.cpp:115-159) over the block. Vectors: y, f0, and
// k2..k6 in a..e, the stage argument in f.
template <class Prob, class R>
__device__ void rkck_wide_system(const WideVecs& V, double t_in, double tEnd_in,
                                 const DevTol& tol, DevStats& st) {
    using namespace ck;
    const int n = V.n;
    double *y = V.y, *f0 = V.f0, *k3 = V.b, *k4 = V.c, *k5 = V.d, *k6 = V.e;
    stats_init(st);
    const R tEnd(tEnd_in);
    R t(t_in);
    const R hMax = fabs_(tEnd - t);
    const R hMin(tol.h_min_floor);
    R h = R(0.5) * fabs_(tEnd - t);
    const R uround(tol.uround), eps(tol.eps), tiny(tol.tiny);
    bool haveF = false;
    AttemptBudget<true> bud;
    bud.init(tol);
#pragma unroll 1
    while (tEnd - t > uround * fabs_(tEnd)) {
        if (bud.spent(st)) break;
        h = fmin_(tEnd - t, h);
        if (!haveF) {  // rejected retries reuse f(t, y) (rkck.cpp:133-137)
            wide_rhs<Prob, R>(V, t, y, f0);
            ++st.rhs_evals;
            haveF = true;
        }
        rkck_wide_stages<Prob, R>(V, t, h, y, f0);  // rkck::step (rkck.cpp:42-64)
        st.rhs_evals += 5;
        st.stages_total += 6;
        // yErr (rkck.cpp:75-76) folded into errorNorm (rkck.cpp:88-98); the
        // max is order-independent (fmax), so a block reduction is exact
        R err(0.0);
        bool nanFlag = false;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const R yErr = h * (R(d1) * R(f0[i]) + R(d3) * R(k3[i]) + R(d4) * R(k4[i]) +
                                R(d5) * R(k5[i]) + R(d6) * R(k6[i]));
            if (!isfinite_(yErr)) nanFlag = true;
            err = fmax_(err, fabs_(yErr / (fabs_(R(y[i])) + fabs_(h * R(f0[i])) + tiny)));
        }
        err = R(block_max(V.red, val(err)));
        nanFlag = block_any(nanFlag);
        err = err / eps;
        R hNew;
        const bool accepted = rkck_adjust(h, err, nanFlag, hMin, hMax, tol, hNew);
        trace_step<true>(tol, threadIdx.x == 0, t, h, 6, err, accepted);
        if (accepted) {
            t += h;
            stats_accept(st, val(h));
            rkck_wide_update<R>(V, h, y, f0);  // yNext (rkck.cpp:74)
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
    __syncthreads();
}

// specrad::powerMethod (spectral_radius.cpp:17-85): v in `v`, f(t, v) in
// `fv`, the warm start / result in `eig`; `tmp` holds the sum terms.
template <class Prob, class R>
__device__ int power_method_wide(const WideVecs& V, R t, const double* y, const double* f0,
                                 double* eig, double* v, double* fv, double* tmp, R hMax,
                                 R& sigmaOut) {
    const int n = V.n;
    constexpr int kItMax = 50;
    const R kUround(2.22e-16);
    const R sqrtU = sqrt_(kUround);
    const R small = R(1.0) / hMax;
    for (int i = threadIdx.x; i < n; i += blockDim.x) tmp[i] = val(R(y[i]) * R(y[i]));
    const R nrmY = sqrt_(block_sum<R>(V.red, tmp, n));
    for (int i = threadIdx.x; i < n; i += blockDim.x) tmp[i] = val(R(eig[i]) * R(eig[i]));
    const R nrmV = sqrt_(block_sum<R>(V.red, tmp, n));
    R dynrm;
    if (nrmY != R(0.0) && nrmV != R(0.0)) {
        dynrm = nrmY * sqrtU;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            v[i] = val(R(y[i]) + R(eig[i]) * (dynrm / nrmV));
    } else if (nrmY != R(0.0)) {
        dynrm = nrmY * sqrtU;
        for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = val(R(y[i]) * (R(1.0) + sqrtU));
    } else if (nrmV != R(0.0)) {
        dynrm = kUround;
        for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = val(R(eig[i]) * (dynrm / nrmV));
    } else {
        dynrm = kUround;
        for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = val(kUround);
    }
    R sigma(0.0);
    int iters = 0;
#pragma unroll 1
    for (int iter = 1; iter <= kItMax; ++iter) {
        wide_rhs<Prob, R>(V, t, v, fv);
        iters = iter;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const R d = R(fv[i]) - R(f0[i]);
            tmp[i] = val(d * d);
        }
        const R diffNrm = sqrt_(block_sum<R>(V.red, tmp, n));
        const R sigmaOld = sigma;
        sigma = diffNrm / dynrm;
        if (iter >= 2 && fabs_(sigma - sigmaOld) <= fmax_(sigma, small) * R(0.01)) break;
        if (diffNrm != R(0.0)) {
            for (int i = threadIdx.x; i < n; i += blockDim.x)
                v[i] = val(R(y[i]) + (R(fv[i]) - R(f0[i])) * (dynrm / diffNrm));
        } else {  // degenerate direction: flip one component about y
            const int ind = iter % n;
            if (threadIdx.x == ind % blockDim.x)
                v[ind] = val(R(y[ind]) - (R(v[ind]) - R(y[ind])));
        }
    }
    sigmaOut = R(1.2) * sigma;
    for (int i = threadIdx.x; i < n; i += blockDim.x) eig[i] = val(R(v[i]) - R(y[i]));
    __syncthreads();
    return iters;
}

// rkc::step (rkc.cpp:82-117) over the block: the s-stage recurrence from y and
// f0 with the stage pair in wA/wB and the stage RHS in fs; returns the vector
// holding y_trial. Coefficients (rkc.cpp:29-69) from the device table for
// s <= kRkcTableMaxS (tab non-null), else the generator.
template <class Prob, class R>
__device__ double* rkc_wide_stages(const WideVecs& V, R t, R h, long long s, R kappa,
                                   const double* tab, const double* y, const double* f0,
                                   double* wA, double* wB, double* fs) {
    const int n = V.n;
    const double* crow = (tab != nullptr && s <= kRkcTableMaxS) ? tab + rkc_table_row(s) : nullptr;
    RkcCoefGen<R> gen;
    R mu1;
    if (crow != nullptr) {
        mu1 = R(crow[0]);
    } else {
        gen.init(s, kappa);
        mu1 = gen.mu1;
    }
    double *wjm1 = wA, *wjm2 = wB;
    {
        const R mu1h = mu1 * h;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            wjm1[i] = val(R(y[i]) + mu1h * R(f0[i]));
    }
#pragma unroll 1
    for (long long j = 2; j <= s; ++j) {
        R muj, nuj, muTj, gTj, cjm1;
        if (crow != nullptr) {
            const double* e = crow + 1 + 5 * (j - 2);
            muj = R(e[0]);
            nuj = R(e[1]);
            muTj = R(e[2]);
            gTj = R(e[3]);
            cjm1 = R(e[4]);
        } else {
            gen.next(j, muj, nuj, muTj, gTj, cjm1);
        }
        wide_rhs<Prob, R>(V, t + cjm1 * h, wjm1, fs);
        const R mujh = muTj * h, gjh = gTj * h;
        if (j == 2) {
            for (int i = threadIdx.x; i < n; i += blockDim.x)
                wjm2[i] = val(R(y[i]) + muj * (R(wjm1[i]) - R(y[i])) + mujh * R(fs[i]) +
                              gjh * R(f0[i]));
        } else {
            for (int i = threadIdx.x; i < n; i += blockDim.x)
                wjm2[i] = val(R(y[i]) + muj * (R(wjm1[i]) - R(y[i])) +
                              nuj * (R(wjm2[i]) - R(y[i])) + mujh * R(fs[i]) + gjh * R(f0[i]));
        }
        double* sw = wjm1;
        wjm1 = wjm2;
        wjm2 = sw;
    }
    return wjm1;
}

// rkc::driver (rkc.cpp:193-281) over the block. Vectors: y, f0, the
// eigenvector in a, the stage pair w_{j-1}/w_{j-2} in b/c, the stage RHS in
// d, the trial RHS in e, sum terms in f. The power method borrows b (v) and
// d (f(v)), which are dead at its call sites.
template <class Prob, class R>
__device__ void rkc_wide_system(const WideVecs& V, double t_in, double tEnd_in,
                                const DevTol& tol, DevStats& st) {
    const int n = V.n;
    double *y = V.y, *f0 = V.f0, *eig = V.a, *wA = V.b, *wB = V.c, *fs = V.d, *ft = V.e,
           *tmp = V.f;
    stats_init(st);
    const R tEnd(tEnd_in);
    R t(t_in);
    const R uround(tol.uround), absTol(tol.abs_tol), relTol(tol.rel_tol), kappa(tol.kappa);
    const R hMax = fabs_(tEnd - t);
    long long mMax = llround(val(sqrt_(relTol / (R(10.0) * uround))));  // rkc.cpp:132-133
    if (mMax < 2) mMax = 2;
    R wsErrOld(0.0), wsHOld(0.0), wsH(0.0), wsSpecRad(0.0);  // Workspace::reset
    R cbErrOld(0.0);
    const R cbrtU = cbrt_(uround);
    long long numStep = 0;
    const R nR = R(static_cast<double>(n));
    AttemptBudget<true> bud;
    bud.init(tol);

    wide_rhs<Prob, R>(V, t, y, f0);  // rkc.cpp:209-212
    ++st.rhs_evals;
    for (int i = threadIdx.x; i < n; i += blockDim.x) eig[i] = f0[i];

    auto estimate = [&]() {
        R sig;
        const int it = power_method_wide<Prob, R>(V, t, y, f0, eig, wA, fs, tmp, hMax, sig);
        wsSpecRad = sig;
        ++st.spec_rad_evals;
        st.rhs_evals += it;
    };
#pragma unroll 1
    while (tEnd - t > uround * fabs_(tEnd)) {
        if (bud.spent(st)) break;
        const R hMin = R(10.0) * uround * fmax_(fabs_(t), hMax);
        if (R(1.1) * wsH >= fabs_(tEnd - t)) wsH = fabs_(tEnd - t);
        if (numStep % 25 == 0) estimate();
        if (wsH < uround) {  // initialStep (rkc.cpp:146-171)
            R h = hMax;
            if (wsSpecRad * h > R(1.0)) h = R(1.0) / wsSpecRad;
            h = fmax_(h, hMin);
            for (int i = threadIdx.x; i < n; i += blockDim.x)
                wA[i] = val(R(y[i]) + h * R(f0[i]));
            wide_rhs<Prob, R>(V, t + h, wA, fs);
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const R est = (R(fs[i]) - R(f0[i])) / (absTol + relTol * fabs_(R(y[i])));
                tmp[i] = val(est * est);
            }
            const R err = h * sqrt_(block_sum<R>(V.red, tmp, n) / nR);
            if (R(0.1) * h < hMax * sqrt_(err))
                h = fmax_(R(0.1) * h / sqrt_(err), hMin);
            else
                h = hMax;
            ++st.rhs_evals;
            wsH = h;
        }
        const long long s = rkc_stage_count(wsSpecRad, mMax, wsH);  // sigma non-finite -> 0
        const R h = wsH;
        // rkc::step (rkc.cpp:82-117)
        double* yTrial = rkc_wide_stages<Prob, R>(V, t, h, s, kappa, tol.rkc_coef, y, f0, wA, wB, fs);
        st.rhs_evals += s - 1;
        st.stages_total += s;
        wide_rhs<Prob, R>(V, t + h, yTrial, ft);  // rkc.cpp:247
        ++st.rhs_evals;
        // errorNorm (rkc.cpp:119-129)
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const R yo(y[i]), yn(yTrial[i]);
            R est = R(0.8) * (yo - yn) + R(0.4) * h * (R(f0[i]) + R(ft[i]));
            est = est / (absTol + relTol * fmax_(fabs_(yo), fabs_(yn)));
            tmp[i] = val(est * est);
        }
        const R err = sqrt_(block_sum<R>(V.red, tmp, n) / nR);
        R hNewRej(0.0);
        trace_step<true>(tol, threadIdx.x == 0, t, h, (int)s, err, err <= R(1.0));
        if (rkc_finish_attempt<R>(err, h, hMin, hMax, uround, cbrtU, tol.p1, st, t, numStep,
                                  wsErrOld, cbErrOld, wsHOld, wsH, hNewRej)) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = yTrial[i];
            double* sw = f0;  // FSAL swap (rkc.cpp:276)
            f0 = ft;
            ft = sw;
            __syncthreads();
        } else {
            estimate();  // rkc.cpp:259
            if (hNewRej < hMin) {  // freeze at the last accepted state (rkc.cpp:260-263)
                st.underflow = 1;
                break;
            }
            wsH = hNewRej;
        }
    }
    // y was always updated in place (V.y); f0/ft swaps only move pointers
    __syncthreads();
}

// One block per system (grid-stride over systems), vectors in shared memory
// (tol.scratch == nullptr) or in this block's slice of tol.scratch.
template <class Prob, class R, int SOLVER>
__global__ void __launch_bounds__(kWideMaxBlock)
    wide_kernel(const double* __restrict__ g_soa, double* __restrict__ y_soa,
                DevStats* __restrict__ stats, long long num, double t, double tEnd, DevTol tol,
                int merge) {
    extern __shared__ double bode_smem[];
    __shared__ double red[33];
    const int n = tol.dim;
    const long long ld = tol.stride > 0 ? tol.stride : num;
    double* base = tol.scratch != nullptr ? tol.scratch + (long long)blockIdx.x * kWideVecs * n
                                          : bode_smem;
    WideVecs V;
    V.y = base;
    V.f0 = base + (long long)n;
    V.a = base + 2LL * n;
    V.b = base + 3LL * n;
    V.c = base + 4LL * n;
    V.d = base + 5LL * n;
    V.e = base + 6LL * n;
    V.f = base + 7LL * n;
    V.n = n;
    V.inv = Prob::inv_dx2(n);
    V.red = red;
    (void)g_soa;
#pragma unroll 1
    for (long long sys = blockIdx.x; sys < num; sys += gridDim.x) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) V.y[i] = y_soa[sys + ld * (long long)i];
        __syncthreads();
        DevStats st;
        if constexpr (SOLVER == 0)
            rkck_wide_system<Prob, R>(V, t, tEnd, tol, st);
        else
            rkc_wide_system<Prob, R>(V, t, tEnd, tol, st);
        for (int i = threadIdx.x; i < n; i += blockDim.x) y_soa[sys + ld * (long long)i] = V.y[i];
        if (stats != nullptr && threadIdx.x == 0) {
            if (merge) {
                DevStats o = stats[sys];
                stats_merge(o, st);
                stats[sys] = o;
            } else {
                stats[sys] = st;
            }
        }
        __syncthreads();  // the vectors are reused by the next system
    }
}

// rkck::integrateFixed (rkck.cpp:168-181) / rkc::integrateFixed (rkc.cpp:290-306)
// for one system per block: numSteps steps of (tEnd - t0) / numSteps, no
// controller. Vectors in shared memory, or in this block's slice of scratch.
template <class Prob, class R, int SOLVER>
__global__ void __launch_bounds__(kWideMaxBlock)
    wide_fixed_kernel(const double* __restrict__ g_soa, double* __restrict__ y_soa, long long num,
                      double t0, double tEnd, long long numSteps, long long stages, double kappa,
                      int n, double* scratch) {
    extern __shared__ double bode_smem[];
    __shared__ double red[33];
    double* base = scratch != nullptr ? scratch + (long long)blockIdx.x * kWideVecs * n : bode_smem;
    WideVecs V;
    V.y = base;
    V.f0 = base + (long long)n;
    V.a = base + 2LL * n;
    V.b = base + 3LL * n;
    V.c = base + 4LL * n;
    V.d = base + 5LL * n;
    V.e = base + 6LL * n;
    V.f = base + 7LL * n;
    V.n = n;
    V.inv = Prob::inv_dx2(n);
    V.red = red;
    (void)g_soa;
    const R h = (R(tEnd) - R(t0)) / R(double(numSteps));  // rkck.cpp:174, rkc.cpp:298
#pragma unroll 1
    for (long long sys = blockIdx.x; sys < num; sys += gridDim.x) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) V.y[i] = y_soa[sys + num * (long long)i];
#pragma unroll 1
        for (long long k = 0; k < numSteps; ++k) {
            const R t = R(t0) + R(double(k)) * h;  // rkck.cpp:176, rkc.cpp:301
            wide_rhs<Prob, R>(V, t, V.y, V.f0);
            if constexpr (SOLVER == 0) {
                rkck_wide_stages<Prob, R>(V, t, h, V.y, V.f0);
                rkck_wide_update<R>(V, h, V.y, V.f0);
            } else {
                const double* yt = rkc_wide_stages<Prob, R>(V, t, h, stages, R(kappa), nullptr, V.y,
                                                            V.f0, V.b, V.c, V.d);
                for (int i = threadIdx.x; i < n; i += blockDim.x) V.y[i] = yt[i];
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) y_soa[sys + num * (long long)i] = V.y[i];
        __syncthreads();
    }
}

}  // namespace bode
