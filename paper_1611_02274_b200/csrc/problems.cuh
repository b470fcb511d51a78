// problems.cuh -- fused device right-hand sides (the paper's user dydt,
// PAPER.md:370, :416), one per reference problem (proj/src/problems.cpp).
//
// A system is owned by a group of L consecutive lanes; lane l holds the C =
// N/L components [l*C, (l+1)*C) of every state-length vector in registers.
// rhs() computes the lane's slice of dy/dt; problems whose RHS couples
// components across lanes (the heat stencil) exchange halos with warp
// shuffles. Expression shapes and accumulation orders follow the reference
// exactly, so with R = xd the result is bitwise the reference's.
#pragma once

#include <type_traits>

#include "arith.cuh"

namespace bode {

// Lane group of L lanes (L divides 32) inside a warp. The shuffles name the
// group's own lanes by default; a warp-uniform caller (every lane of the warp
// reaches every shuffle, as the RKC driver guarantees) passes full = true, and
// the constant full mask lets ptxas drop its per-shuffle convergence check
// (MATCH.ANY / REDUX / VOTE and a divergent-path branch).
template <int L>
struct Group {
    int lane;       // 0..L-1
    unsigned mask;  // the lanes taking part in each shuffle
    __device__ __forceinline__ explicit Group(bool full = false) {
        const int wl = threadIdx.x & 31;
        lane = wl & (L - 1);
        mask = (L == 32 || full) ? 0xffffffffu : (((1u << L) - 1u) << (wl & ~(L - 1)));
    }
    // value held by group lane `src`
    __device__ __forceinline__ double from(double v, int src) const {
        return __shfl_sync(mask, v, src, L);
    }
    __device__ __forceinline__ double from_prev(double v) const {  // lane-1
        return __shfl_up_sync(mask, v, 1, L);
    }
    __device__ __forceinline__ double from_next(double v) const {  // lane+1
        return __shfl_down_sync(mask, v, 1, L);
    }
    __device__ __forceinline__ double max_all(double v) const {  // fmax over lanes
#pragma unroll
        for (int o = L / 2; o > 0; o /= 2) v = fmax(v, __shfl_xor_sync(mask, v, o, L));
        return v;
    }
    // any lane of this group (the vote spans `mask`, the answer the group only)
    __device__ __forceinline__ bool any(bool b) const {
        const unsigned own = (L == 32) ? 0xffffffffu
                                       : (((1u << L) - 1u) << ((threadIdx.x & 31) & ~(L - 1)));
        return (__ballot_sync(mask, b) & own) != 0u;
    }
};

template <>
struct Group<1> {
    int lane = 0;
    unsigned mask = 0u;
    __device__ __forceinline__ explicit Group(bool = false) {}
    __device__ __forceinline__ double from(double v, int) const { return v; }
    __device__ __forceinline__ double from_prev(double v) const { return v; }
    __device__ __forceinline__ double from_next(double v) const { return v; }
    __device__ __forceinline__ double max_all(double v) const { return v; }
    __device__ __forceinline__ bool any(bool b) const { return b; }
};

template <class R, int L>
__device__ __forceinline__ R grp_from(const Group<L>& G, R v, int src) {
    return R(G.from(val(v), src));
}

// Sequential sum in global component order: lane 0 sums its C terms, hands
// the partial to lane 1, ... exactly the reference's `sum += term` loop
// (rkc.cpp:122-127, spectral_radius.cpp:11-13). Result valid on every lane.
template <class R, int L, int C>
__device__ __forceinline__ R seq_sum(const Group<L>& G, const R (&terms)[C], R init) {
    if constexpr (L == 1) {
        R s = init;
#pragma unroll
        for (int c = 0; c < C; ++c) s = s + terms[c];
        return s;
    } else {
        R s = init;
#pragma unroll 1
        for (int k = 0; k < L; ++k) {
            if (G.lane == k) {
#pragma unroll
                for (int c = 0; c < C; ++c) s = s + terms[c];
            }
            s = R(G.from(val(s), k));
        }
        return s;
    }
}

// Two independent sequential sums advanced together (each in its own
// component order, so each is bitwise seq_sum's): the chains interleave, and
// the pair costs one chain's latency.
template <class R, int L, int C>
__device__ __forceinline__ void seq_sum2(const Group<L>& G, const R (&a)[C], const R (&b)[C],
                                         R& sa, R& sb) {
    if constexpr (L == 1) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            sa = sa + a[c];
            sb = sb + b[c];
        }
    } else {
#pragma unroll 1
        for (int k = 0; k < L; ++k) {
            if (G.lane == k) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    sa = sa + a[c];
                    sb = sb + b[c];
                }
            }
            sa = R(G.from(val(sa), k));
            sb = R(G.from(val(sb), k));
        }
    }
}

// -------------------------------------------------------------------------
// Pleiades (problems.cpp:9-37): N = 28, masses m_i = i + 1, pairs i<j with
// i outer, j inner; action/reaction share one distance evaluation.
struct Pleiades {
    static constexpr int N = 28, P = 0;
    static constexpr bool second_order = true;  // out[0..14) = w[14..28) (problems.cpp:17)
    static constexpr const char* name = "pleiades";
    // Accelerations a(q) for positions q = (x_1..x_7, y_1..y_7): the out[14..27]
    // half of the reference RHS, accumulated in the reference's order.
    template <class R>
    __device__ __forceinline__ static void accel(R, const R* w, const R*, R* a) {
        // EXACT: 1/(r2 sqrt(r2)) for all pairs first, straight-line (arith.cuh
        // sqrt_rn_bf / rcp_rn_bf), with one cold fallback to the intrinsics
        double inv[21];
        if constexpr (is_exact<R>::value) {
            bool ok = true;
#pragma unroll
            for (int p = 0, i = 0; i < 7; ++i)
#pragma unroll
                for (int j = i + 1; j < 7; ++j, ++p) {
                    const R dx = w[j] - w[i];
                    const R dy = w[7 + j] - w[7 + i];
                    const double r2 = val(dx * dx + dy * dy);
                    const double d = __dmul_rn(r2, sqrt_rn_bf(r2));
                    ok = ok & r3_in_safe_range(r2);
                    inv[p] = rcp_rn_bf(d);
                }
            if (!ok) {  // rare: some operand outside [2^-400, 2^400] (or NaN/Inf)
#pragma unroll
                for (int p = 0, i = 0; i < 7; ++i)
#pragma unroll
                    for (int j = i + 1; j < 7; ++j, ++p) {
                        const R dx = w[j] - w[i];
                        const R dy = w[7 + j] - w[7 + i];
                        const R r2 = dx * dx + dy * dy;
                        inv[p] = val(R(1.0) / (r2 * sqrt_(r2)));
                    }
            }
        }
#pragma unroll
        for (int i = 0; i < 14; ++i) a[i] = R(0.0);
#pragma unroll
        for (int p = 0, i = 0; i < 7; ++i) {
#pragma unroll
            for (int j = i + 1; j < 7; ++j, ++p) {
                const R dx = w[j] - w[i];
                const R dy = w[7 + j] - w[7 + i];
                const double mi = double(i + 1);
                const double mj = double(j + 1);
                if constexpr (is_exact<R>::value) {
                    const R invR3(inv[p]);
                    a[i] += R(mj) * dx * invR3;
                    a[7 + i] += R(mj) * dy * invR3;
                    a[j] -= R(mi) * dx * invR3;
                    a[7 + j] -= R(mi) * dy * invR3;
                } else {
                    const R r2 = dx * dx + dy * dy;
                    const double invR3 = rsqrt3_fast(val(r2));
                    const double ax = val(dx) * invR3;
                    const double ay = val(dy) * invR3;
                    a[i] += mj * ax;
                    a[7 + i] += mj * ay;
                    a[j] -= mi * ax;
                    a[7 + j] -= mi * ay;
                }
            }
        }
    }
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R, const R (&w)[N],
                                               const R*, R (&out)[N]) {
        static_assert(L == 1, "Pleiades couples all components: one lane per system");
#pragma unroll
        for (int i = 0; i < 14; ++i) out[i] = w[14 + i];
        accel<R>(R(0.0), w, nullptr, out + 14);
    }
};

// Second-order systems y = (q, v), q' = v, v' = a(t, q; g): derive from this
// with the problem struct itself as D and M = dim(q), and provide
//   template <class R> __device__ static void accel(R t, const R* q, const R* g, R* a);
// RKCK then runs the Nystrom kernels (rkck_nystrom.cuh: the reference's step
// on velocity-copy storage under EXACT, the Runge-Kutta-Nystrom form under
// FAST); RKC and the fixed-step harnesses use the rhs() below, which is the
// reference-style full right-hand side (velocities first, then a).
template <class D, int M_, int P_ = 0>
struct SecondOrderProblem {
    static constexpr int N = 2 * M_, P = P_;
    static constexpr bool second_order = true;
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R t, const R (&w)[N / L],
                                               const R* g, R (&out)[N / L]) {
        static_assert(L == 1, "second-order problems run one lane per system");
#pragma unroll
        for (int i = 0; i < M_; ++i) out[i] = w[M_ + i];
        D::template accel<R>(t, w, g, out + M_);
    }
};

// Heat equation, method of lines (problems.cpp:94-115): N = n interior
// points, (u[i-1] - 2 u[i] + u[i+1]) / dx^2 with zero Dirichlet boundaries.
template <int NN>
struct Heat {
    static constexpr int N = NN, P = 0;
    static constexpr const char* name = "heat";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>& G, R, const R (&u)[N / L],
                                               const R*, R (&out)[N / L]) {
        constexpr int C = N / L;
        const double dx = 1.0 / (NN + 1);
        const double inv = 1.0 / (dx * dx);
        // halo values from the neighbouring lanes (unused at the boundaries)
        const R left = R(G.from_prev(val(u[C - 1])));
        const R right = R(G.from_next(val(u[0])));
        const bool first = G.lane == 0, last = G.lane == L - 1;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const R um = (c > 0) ? u[c - 1] : left;
            const R up = (c < C - 1) ? u[c + 1] : right;
            if (c == 0 && first)
                out[c] = (R(-2.0) * u[c] + up) * R(inv);
            else if (c == C - 1 && last)
                out[c] = (um - R(2.0) * u[c]) * R(inv);
            else
                out[c] = (um - R(2.0) * u[c] + up) * R(inv);
        }
    }
};

// Run-time dimension on the lane-group kernels: a problem with
// `runtime_dim = true` has the compile-time capacity N (lane groups of N/L
// components) and integrates the first n <= N components, n = tol.dim. The
// kernel hands n and the problem's constant to rhs() in g[0] and g[1] (the
// problem has no parameters of its own); the components from n to N are
// padding that stays exactly +0.0, which leaves every reference sum and max
// bitwise unchanged (a +0.0 term adds nothing to a sum of squares or a
// max-norm), so the results are the unpadded reference's.
template <class P, class = void>
struct is_runtime_dim : std::false_type {};
template <class P>
struct is_runtime_dim<P, decltype((void)P::runtime_dim)> : std::bool_constant<P::runtime_dim> {};
// the system's dimension (the divisor of the RMS norms, rkc.cpp:128, :164;
// the flip index of the power method, spectral_radius.cpp:76)
template <class P, class R>
__device__ __forceinline__ int dim_of(const R* g) {
    if constexpr (is_runtime_dim<P>::value)
        return (int)val(g[0]);
    else
        return P::N;
}

// heatEquation(n) (problems.cpp:94-115) for any n <= CAP on CAP-component lane
// groups: g[0] = n, g[1] = 1/dx^2 formed as the reference does, in IEEE double.
template <int CAP>
struct HeatPad {
    static constexpr int N = CAP, P = 0, PG = 2;
    static constexpr bool runtime_dim = true;
    static constexpr const char* name = "heat";
    __device__ __forceinline__ static void params(int n, double* g) {
        g[0] = double(n);
        const double dx = __ddiv_rn(1.0, double(n + 1));
        g[1] = __ddiv_rn(1.0, __dmul_rn(dx, dx));
    }
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>& G, R, const R (&u)[N / L],
                                               const R* g, R (&out)[N / L]) {
        constexpr int C = N / L;
        const int n = (int)val(g[0]);
        const R inv = g[1];
        const R left = R(G.from_prev(val(u[C - 1])));
        const R right = R(G.from_next(val(u[0])));
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int i = G.lane * C + c;
            const R um = (c > 0) ? u[c - 1] : left;
            const R up = (c < C - 1) ? u[c + 1] : right;
#ifndef BODE_HEATPAD_BRANCHY
            // The boundary and padding cases by selects, not branches (which
            // diverge inside every lane group: i depends on the lane and the
            // run-time n). Same IEEE operations per case as the reference:
            // R(-2.0) * u == -(2u) exactly, so i = 0 is -(2u) + up, the last
            // point um - 2u, the interior (um - 2u) + up.
            const R u2 = R(2.0) * u[c];
            const R a = (i == 0) ? -u2 : um - u2;
            const R b = (i == n - 1) ? a : a + up;
            out[c] = (i >= n) ? R(0.0) : b * inv;
#else
            if (i >= n)
                out[c] = R(0.0);
            else if (i == 0)
                out[c] = (R(-2.0) * u[c] + up) * inv;
            else if (i == n - 1)
                out[c] = (um - R(2.0) * u[c]) * inv;
            else
                out[c] = (um - R(2.0) * u[c] + up) * inv;
#endif
        }
    }
};

// dy/dt = -g0 y (problems.cpp:134-144)
struct ExpDecay {
    static constexpr int N = 1, P = 1;
    static constexpr const char* name = "expdecay";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R, const R (&y)[1],
                                               const R* g, R (&out)[1]) {
        out[0] = -g[0] * y[0];
    }
};

// (q, p)' = (p, -q) (problems.cpp:146-156)
struct Harmonic {
    static constexpr int N = 2, P = 0;
    static constexpr const char* name = "harmonic";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R, const R (&y)[2],
                                               const R*, R (&out)[2]) {
        out[0] = y[1];
        out[1] = -y[0];
    }
};

// Calibration problems of the reference test suites.
template <int NN>
struct Zero {  // test_batch.cpp:80-89
    static constexpr int N = NN, P = 0;
    static constexpr const char* name = "zero";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R, const R (&)[N / L],
                                               const R*, R (&out)[N / L]) {
#pragma unroll
        for (int c = 0; c < N / L; ++c) out[c] = R(0.0);
    }
};

struct Riccati {  // y' = y^2 (test_rkck.cpp:28)
    static constexpr int N = 1, P = 0;
    static constexpr const char* name = "riccati";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R, const R (&y)[1],
                                               const R*, R (&out)[1]) {
        out[0] = y[0] * y[0];
    }
};

template <int NN>
struct Diag {  // y_i' = g_i y_i (test_specrad.cpp:16-24)
    static constexpr int N = NN, P = NN;
    static constexpr const char* name = "diag";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>& G, R, const R (&y)[N / L],
                                               const R* g, R (&out)[N / L]) {
#pragma unroll
        for (int c = 0; c < N / L; ++c) out[c] = g[G.lane * (N / L) + c] * y[c];
    }
};

template <int NN>
struct Const {  // y' = 1 (test_rkck.cpp:26)
    static constexpr int N = NN, P = 0;
    static constexpr const char* name = "const";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R, const R (&)[N / L],
                                               const R*, R (&out)[N / L]) {
#pragma unroll
        for (int c = 0; c < N / L; ++c) out[c] = R(1.0);
    }
};

struct SinT {  // y' = sin(t) y (test_rkck.cpp:220-230)
    static constexpr int N = 1, P = 0;
    static constexpr const char* name = "sint";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>&, R t, const R (&y)[1],
                                               const R*, R (&out)[1]) {
        out[0] = sin_(t) * y[0];
    }
};

}  // namespace bode
