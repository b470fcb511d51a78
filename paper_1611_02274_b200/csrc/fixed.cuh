// fixed.cuh -- fixed-step, controller-free harnesses:
// rkck::integrateFixed (rkck.cpp:168-181) and rkc::integrateFixed
// (rkc.cpp:290-306), one system per lane group. The order-of-convergence
// acceptance criterion (acceptance.cpp:92-124: slopes 5 +- 0.3, 2 +- 0.2)
// runs on them, validating the device stage arithmetic independently of the
// step-size controllers.
#pragma once

#include "rkc.cuh"

namespace bode {

// rkck::step (rkck.cpp:34-78) with stage storage in registers; returns yNext.
template <class P, class R, int L>
__device__ __forceinline__ void rkck_fixed_step(const Group<L>& G, R t, R (&y)[P::N / L],
                                                const R* g, R h) {
    constexpr int C = P::N / L;
    using namespace ck;
    R f0[C], k2[C], k3[C], k4[C], k5[C], k6[C], arg[C];
    P::template rhs<R, L>(G, t, y, g, f0);
#pragma unroll
    for (int c = 0; c < C; ++c) arg[c] = y[c] + h * R(b21) * f0[c];
    P::template rhs<R, L>(G, t + R(a2) * h, arg, g, k2);
#pragma unroll
    for (int c = 0; c < C; ++c) arg[c] = y[c] + h * (R(b31) * f0[c] + R(b32) * k2[c]);
    P::template rhs<R, L>(G, t + R(a3) * h, arg, g, k3);
#pragma unroll
    for (int c = 0; c < C; ++c)
        arg[c] = y[c] + h * (R(b41) * f0[c] + R(b42) * k2[c] + R(b43) * k3[c]);
    P::template rhs<R, L>(G, t + R(a4) * h, arg, g, k4);
#pragma unroll
    for (int c = 0; c < C; ++c)
        arg[c] = y[c] + h * (R(b51) * f0[c] + R(b52) * k2[c] + R(b53) * k3[c] + R(b54) * k4[c]);
    P::template rhs<R, L>(G, t + R(a5) * h, arg, g, k5);
#pragma unroll
    for (int c = 0; c < C; ++c)
        arg[c] = y[c] + h * (R(b61) * f0[c] + R(b62) * k2[c] + R(b63) * k3[c] + R(b64) * k4[c] +
                             R(b65) * k5[c]);
    P::template rhs<R, L>(G, t + R(a6) * h, arg, g, k6);
#pragma unroll
    for (int c = 0; c < C; ++c)
        y[c] = y[c] + h * (R(c1) * f0[c] + R(c3) * k3[c] + R(c4) * k4[c] + R(c6) * k6[c]);
}

// rkc::step (rkc.cpp:82-117) with fixed s, coefficients from RkcCoefGen.
template <class P, class R, int L>
__device__ __forceinline__ void rkc_fixed_step(const Group<L>& G, R t, R (&y)[P::N / L],
                                               const R* g, R h, long long s, R kappa) {
    constexpr int C = P::N / L;
    R f0[C], wa[C], wb[C];
    P::template rhs<R, L>(G, t, y, g, f0);
    RkcCoefGen<R> gen;
    gen.init(s, kappa);
    const R mu1h = gen.mu1 * h;
#pragma unroll
    for (int c = 0; c < C; ++c) wa[c] = y[c] + mu1h * f0[c];
    bool inA = true;
#pragma unroll 1
    for (long long j = 2; j <= s; ++j) {
        R muj, nuj, muTj, gTj, cjm1;
        gen.next(j, muj, nuj, muTj, gTj, cjm1);
        const R tj = t + cjm1 * h;
        R f[C];
        R(&src)[C] = inA ? wa : wb;
        R(&dst)[C] = inA ? wb : wa;
        P::template rhs<R, L>(G, tj, src, g, f);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (j == 2)
                dst[c] = y[c] + muj * (src[c] - y[c]) + (muTj * h) * f[c] + (gTj * h) * f0[c];
            else
                dst[c] = y[c] + muj * (src[c] - y[c]) + nuj * (dst[c] - y[c]) + (muTj * h) * f[c] +
                         (gTj * h) * f0[c];
        }
        inA = !inA;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = inA ? wa[c] : wb[c];
}

template <class P, class R, int L, int SOLVER>
__global__ void __launch_bounds__(kMaxBlock)
    fixed_kernel(const double* __restrict__ g_soa, double* __restrict__ y_soa, long long num,
                 double t0, double tEnd, long long numSteps, long long stages, double kappa) {
    constexpr int C = P::N / L;
    constexpr int PP = P::P > 0 ? P::P : 1;
    const long long sys = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / L;
    if (sys >= num) return;
    Group<L> G;
    R y[C], g[PP];
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = R(y_soa[sys + num * (long long)(G.lane * C + c)]);
#pragma unroll
    for (int p = 0; p < PP; ++p) g[p] = R(P::P > 0 ? g_soa[sys + num * (long long)p] : 0.0);
    const R h = (R(tEnd) - R(t0)) / R(double(numSteps));  // rkck.cpp:174, rkc.cpp:298
#pragma unroll 1
    for (long long k = 0; k < numSteps; ++k) {
        const R t = R(t0) + R(double(k)) * h;  // rkck.cpp:176, rkc.cpp:301
        if constexpr (SOLVER == 0)
            rkck_fixed_step<P, R, L>(G, t, y, g, h);
        else
            rkc_fixed_step<P, R, L>(G, t, y, g, h, stages, R(kappa));
    }
#pragma unroll
    for (int c = 0; c < C; ++c) y_soa[sys + num * (long long)(G.lane * C + c)] = val(y[c]);
}

}  // namespace bode
