// rkc.cuh -- adaptive Runge-Kutta-Chebyshev integration (with the
// Jacobian-free power-method spectral radius) of one system per lane group.
//
// Follows proj/src/rkc.cpp: chebyshevEval (:10-27), coefficients (:29-69),
// step (:82-117), errorNorm (:119-129), stageCount (:131-144), initialStep
// (:146-171), nextStepAccepted/Rejected (:173-191), driver (:193-281) and
// proj/src/spectral_radius.cpp powerMethod (:17-85).
//
// Differences in *form* only (results are bitwise the reference's with R=xd):
//  * Stage coefficients come from a per-device table (s <= kRkcTableMaxS)
//    filled once by RkcCoefGen, the same generator that runs on the fly for
//    larger s: it runs the Chebyshev recurrence alongside the stages. The
//    reference evaluates chebyshevEval(j, x) from scratch for each j with the
//    same loop, so the j-th iterate is the same double; omega1 needs T'_s and
//    T''_s, obtained by a scalar pre-pass of s iterations.
//  * The driver loop is a small state machine (TOP -> [SPECRAD] -> ATTEMPT,
//    reject -> SPECRAD -> REJECT_TAIL) so the power method, the initial step
//    and the stage recurrence each have one call site in the kernel. The
//    event order per system is exactly the reference's. The loop is
//    warp-uniform: each phase runs for the whole warp when any group needs
//    it, so the lane-group shuffles use the full warp mask.
//  * Sums that the reference accumulates sequentially (error norm, 2-norms)
//    stay sequential in component order across the lane group (seq_sum).
#pragma once

#include "rkck.cuh"

namespace bode {

// Phase timing (tools/phase_probe.cu builds with BODE_PHASE_TIMING): clock64()
// deltas per rkc_system phase, summed over lane groups into g_phase[0..4] =
// power method, initial step, stage loop, f_trial + error norm, controller.
#ifdef BODE_PHASE_TIMING
__device__ unsigned long long* g_phase = nullptr;
#define BODE_PHASE_DECL long long ph_acc[5] = {0, 0, 0, 0, 0}, ph_t = 0, ph_last = -1;
#define BODE_PHASE_MARK(k) do { const long long n_ = clock64(); if ((k) >= 0) ph_acc[k] += n_ - ph_t; ph_t = n_; } while (0)
#define BODE_PHASE_CTRL_BEGIN ph_last = clock64();
#define BODE_PHASE_CTRL_END if (ph_last >= 0) { ph_acc[4] += clock64() - ph_last; ph_last = -1; }
#define BODE_PHASE_FLUSH if (g_phase && G.lane == 0) for (int k_ = 0; k_ < 5; ++k_) atomicAdd(&g_phase[k_], (unsigned long long)ph_acc[k_]);
#else
#define BODE_PHASE_DECL
#define BODE_PHASE_MARK(k)
#define BODE_PHASE_CTRL_BEGIN
#define BODE_PHASE_CTRL_END
#define BODE_PHASE_FLUSH
#endif

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

// Stage coefficients of rkc::coefficients (rkc.cpp:29-69), produced stage by
// stage: init() computes omega0, omega1 (a pre-pass of s Chebyshev steps) and
// muTilde_1; next(j) yields mu_j, nu_j, muTilde_j, gammaTilde_j and the node
// c_{j-1} used by stage j. chebyshevEval(j, x) (rkc.cpp:10-27) restarts the
// same recurrence for every j, so the j-th iterate here is the same double.
template <class R>
struct RkcCoefGen {
    R omega0, omega1, b1, mu1;
    Cheb<R> Tm2, Tm1, T2;
    R bm1, bm2, am1, cjm1, b2;
    long long s;
    __device__ __forceinline__ void init(long long s_, R kappa) {
        s = s_;
        omega0 = R(1.0) + kappa / (R(double(s)) * R(double(s)));
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
        b1 = R(1.0) / omega0;
        mu1 = b1 * omega1;
        Tm2 = Cheb<R>{R(1.0), R(0.0), R(0.0)};
        Tm1 = Cheb<R>{omega0, R(1.0), R(0.0)};
        T2 = cheb_next(Tm1, Tm2, omega0);
        b2 = T2.dd / (T2.d * T2.d);
        bm1 = b1;
        bm2 = b2;  // b_0 = b_2 (rkc.cpp:50), only reached through nu_2 (unused)
        // c_1 = c_2 / (4 omega0), c_2 interior unless s == 2 (then c_2 = c_s = 1)
        const R c2 = (s > 2) ? omega1 * T2.dd / T2.d : R(1.0);
        cjm1 = c2 / (R(4.0) * omega0);
        am1 = R(1.0) - b1 * Tm1.T;  // a_1
    }
    __device__ __forceinline__ void next(long long j, R& muj, R& nuj, R& muTj, R& gTj, R& cout) {
        const Cheb<R> Tj = (j == 2) ? T2 : cheb_next(Tm1, Tm2, omega0);
        const R bj = (j == 2) ? b2 : Tj.dd / (Tj.d * Tj.d);
        muj = R(2.0) * bj * omega0 / bm1;
        nuj = -bj / bm2;
        muTj = R(2.0) * bj * omega1 / bm1;
        gTj = -am1 * muTj;
        cout = cjm1;
        // advance to j+1: c_j (interior for j < s), a_j, b's, T's
        cjm1 = (j < s) ? omega1 * Tj.dd / Tj.d : R(1.0);
        am1 = R(1.0) - bj * Tj.T;
        bm2 = bm1;
        bm1 = bj;
        Tm2 = Tm1;
        Tm1 = Tj;
    }
};

// Shared-memory row per lane: the eigenvector, f0, the lane's stats and (with
// kRkcYInSmem) the state y (3C + 8 doubles, odd stride). The stats are touched a few times per attempt;
// keeping their 15 registers out of the stage loop removes most spills at
// the 128-register cap.
// Lane groups (L > 1) add C doubles of scratch for the sequential sums
// (rkc_seq_sum): each lane posts its terms there for its group.
// Lane groups also keep the controller scalars that live across the whole
// window but are touched once per attempt (kRkcCtrl doubles: cbrt(errOld),
// hOld, the rejected step, the spectral radius, cbrt(uround)) in the row, so
// they hold no registers (or spill slots) through the stage loop.
#ifndef BODE_RKC_CTRL_SMEM
#define BODE_RKC_CTRL_SMEM 1
#endif
constexpr int kRkcCtrl = BODE_RKC_CTRL_SMEM ? 5 : 0;
template <int C, int L = 1>
__host__ __device__ constexpr int kRkcSmemStride() {
    return ((L > 1 ? 4 : 3) * C + 8 + (L > 1 ? kRkcCtrl : 0)) | 1;
}
template <int C>
__host__ __device__ constexpr int kRkcTermsOffset() { return 3 * C + 8; }
template <int C>
__host__ __device__ constexpr int kRkcCtrlOffset() { return 4 * C + 8; }

// Per-device coefficient table for s = 2..kRkcTableMaxS: row(s) holds
// muTilde_1 followed by (mu_j, nu_j, muTilde_j, gammaTilde_j, c_{j-1}) for
// j = 2..s, generated by RkcCoefGen itself (bitwise the on-the-fly values).
constexpr long long kRkcTableMaxS = 160;
__host__ __device__ constexpr long long rkc_table_row(long long s) {
    // sum over s' = 2..s-1 of (1 + 5 (s' - 1))
    return (s - 2) + 5 * ((s - 2) * (s - 1) / 2);
}
constexpr long long kRkcTableDoubles = rkc_table_row(kRkcTableMaxS + 1);

template <class R>
__global__ void rkc_coef_table_kernel(double* tab, double kappa) {
    const long long s = 2 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s > kRkcTableMaxS) return;
    RkcCoefGen<R> gen;
    gen.init(s, R(kappa));
    double* row = tab + rkc_table_row(s);
    row[0] = val(gen.mu1);
    for (long long j = 2; j <= s; ++j) {
        R muj, nuj, muTj, gTj, cj;
        gen.next(j, muj, nuj, muTj, gTj, cj);
        double* e = row + 1 + 5 * (j - 2);
        e[0] = val(muj);
        e[1] = val(nuj);
        e[2] = val(muTj);
        e[3] = val(gTj);
        e[4] = val(cj);
    }
}

// Stage coefficients for s > kRkcTableMaxS: a non-inlined generator whose
// state lives in local memory fills kRkcGenChunk stages at a time into a
// local buffer, so this rare path holds no registers in the hot stage loop.
constexpr int kRkcGenChunk = 16;
template <class R>
__device__ __noinline__ void rkc_gen_start(RkcCoefGen<R>* gen, long long s, double kappa,
                                           double* mu1) {
    gen->init(s, R(kappa));
    *mu1 = val(gen->mu1);
}
template <class R>
__device__ __noinline__ void rkc_gen_chunk(RkcCoefGen<R>* gen, long long j0, long long j1,
                                           double* out) {
    for (long long j = j0; j <= j1; ++j) {
        R muj, nuj, muTj, gTj, cj;
        gen->next(j, muj, nuj, muTj, gTj, cj);
        double* e = out + 5 * (j - j0);
        e[0] = val(muj);
        e[1] = val(nuj);
        e[2] = val(muTj);
        e[3] = val(gTj);
        e[4] = val(cj);
    }
}

// f0 = f(t, y) storage for the RKC driver: registers, or this lane's
// shared-memory row (one conflict-free load per element per stage).
constexpr bool kRkcF0InSmem = true;
// y between the window's entry and exit: in the lane's shared-memory row (for
// slices of >= 4 components), so the stage loop's registers go to the two
// stage vectors. Measured: Brusselator +4%, heat64 neutral at 128 registers
// (+6% at 96); for expDecay (1 component) registers are 3% faster.
constexpr bool kRkcYInSmem = true;
template <class R, int C, bool SMEM>
struct F0Store;
template <class R, int C>
struct F0Store<R, C, false> {
    R v[C];
    __device__ __forceinline__ explicit F0Store(double*) {}
    __device__ __forceinline__ R operator[](int c) const { return v[c]; }
    __device__ __forceinline__ void set(int c, R x) { v[c] = x; }
};
template <class R, int C>
struct F0Store<R, C, true> {
    double* p;
    __device__ __forceinline__ explicit F0Store(double* row) : p(row) {}
    __device__ __forceinline__ R operator[](int c) const { return R(p[c]); }
    __device__ __forceinline__ void set(int c, R x) { p[c] = val(x); }
};

// out[c] = num(c) / den(c) for the lane's C components. EXACT: IEEE
// division; FAST: reciprocal multiply.
constexpr bool kRkcStraightDiv = true;
// ZERO_OK (run-time-dimension problems): +0 numerators, the padding, stay on
// the straight-line path (arith.cuh div_rn_nv).
template <class R, int C, bool ZERO_OK = false, class Num, class Den>
__device__ __forceinline__ void elementwise_quotients(Num num, Den den, R (&out)[C]) {
    if constexpr (is_exact<R>::value && kRkcStraightDiv) {
        // straight-line quotients (arith.cuh div_rn_nv: the intrinsic's own fast
        // path), so the C divisions interleave; one cold fallback to the
        // intrinsic if any of them would leave its fast path
        double a[C], b[C];
        bool ok = true;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            a[c] = val(num(c));
            b[c] = val(den(c));
            bool fast;
            const double q = div_rn_nv(a[c], b[c], fast);
            ok = ok && fast;
            out[c] = R(q);
        }
        if constexpr (ZERO_OK) {
            // a lane holding padding (+0 numerators) lands here every time:
            // accept +0 / b in this cold re-test rather than in the loop above,
            // which leaves lanes without padding exactly the plain code
            if (!ok) {
                ok = true;
#pragma unroll
                for (int c = 0; c < C; ++c)
                    ok = ok && (div_fast_path(a[c], b[c], val(out[c])) || div_zero_num(a[c], b[c]));
            }
        }
        if (!ok) {
#pragma unroll
            for (int c = 0; c < C; ++c) out[c] = R(__ddiv_rn(a[c], b[c]));
        }
    } else if constexpr (is_exact<R>::value) {
        // IEEE intrinsic: its out-of-line slow path splits the code around each
        // division
#pragma unroll
        for (int c = 0; c < C; ++c) out[c] = num(c) / den(c);
    } else {
#pragma unroll
        for (int c = 0; c < C; ++c) out[c] = num(c) * rcp_fast(val(den(c)));
    }
}

// The reference's sequential sums (rkc.cpp:122-127, spectral_radius.cpp:11-13)
// for a lane group: seq_sum's shuffle hand-off. (Measured alternatives, all
// slower: lane 0 running the chain from shared memory, -4%; a shared-memory
// hand-off with __syncwarp, -5%; gathering every term by shuffles, -18%.)
// The RKC sums of squares (error norm rkc.cpp:122-127, initial step
// :160-164, power-method norm spectral_radius.cpp:11-13).
//  EXACT, lane groups: the reference's sequential order. Each lane posts its C
//   terms to its shared-memory scratch, and every lane of the group runs the
//   whole N-term chain over the group's scratch (broadcast loads, issued
//   ahead of the adds), so the chain carries no shuffle hand-offs.
//  FAST: pairwise within the lane, then a butterfly across the group. IEEE
//   addition commutes, so every lane ends with the same value.
#ifndef BODE_RKC_SUM
#define BODE_RKC_SUM 1
#endif
template <class R, int L, int C>
__device__ __forceinline__ R rkc_seq_sum(const Group<L>& G, const R (&terms)[C], R init) {
    if constexpr (L == 1 || BODE_RKC_SUM == 0) {
        return seq_sum<R, L, C>(G, terms, init);
    } else if constexpr (is_exact<R>::value && BODE_RKC_SUM != 2) {  // 2: experiment only (not bitwise)
        extern __shared__ double bode_smem[];
        constexpr int S = kRkcSmemStride<C, L>();
        double* mine = bode_smem + threadIdx.x * S + kRkcTermsOffset<C>();
#pragma unroll
        for (int c = 0; c < C; ++c) mine[c] = val(terms[c]);
        __syncwarp();
        const double* grp = bode_smem + (threadIdx.x & ~(L - 1)) * S + kRkcTermsOffset<C>();
        R s = init;
#pragma unroll
        for (int k = 0; k < L; ++k)
#pragma unroll
            for (int c = 0; c < C; ++c) s = s + R(grp[k * S + c]);
        __syncwarp();  // the scratch is rewritten by the next sum
        return s;
    } else {
        R part[C];
#pragma unroll
        for (int c = 0; c < C; ++c) part[c] = terms[c];
#pragma unroll
        for (int w = 1; w < C; w *= 2)
#pragma unroll
            for (int c = 0; c + w < C; c += 2 * w) part[c] = part[c] + part[c + w];
        R s = part[0];
#pragma unroll
        for (int o = 1; o < L; o *= 2) s = s + R(__shfl_xor_sync(0xffffffffu, val(s), o, L));
        return init + s;
    }
}

// For lane groups (L > 1) every lane of the warp reaches every shuffle of the
// driver below (see rkc_system); this is the warp-wide vote that keeps its
// phases uniform. With one lane per system there are no shuffles and each
// lane branches on its own state.
template <int L>
__device__ __forceinline__ bool phase_any(bool b) {
    if constexpr (L > 1)
        return __any_sync(0xffffffffu, b);
    else
        return b;
}

// x / N for the mean in the RMS norms (rkc.cpp:128, :164). For N a power of
// two, x * 2^-k rounds the same real number, so the product is bitwise the
// quotient (subnormals, infinities and NaN included) without a division.
template <int N, class R>
__device__ __forceinline__ R div_by_dim_ct(R x) {
    if constexpr (N == 1)
        return x;
    else if constexpr ((N & (N - 1)) == 0)
        return x * R(1.0 / N);
    else
        return x / R(double(N));
}
// x / n for the system's dimension: compile-time, or the run-time n of a
// padded problem (an IEEE division, as the reference's)
template <class P, class R>
__device__ __forceinline__ R div_by_dim(R x, const R* g) {
    if constexpr (is_runtime_dim<P>::value)
        return x / R(double(dim_of<P>(g)));
    else
        return div_by_dim_ct<P::N>(x);
}

// Power method (spectral_radius.cpp:17-85) for the groups with `on` set; the
// other groups of the warp run alongside on their own state and discard the
// result. Returns sigma (with the 1.2 safety factor) and the number of
// iterations (= RHS evaluations); eig is the warm start on entry and v - y
// on exit.
template <class P, class R, int L, class Y, class F0>
__device__ __forceinline__ int power_method(const Group<L>& G, bool on, R t, const Y& y,
                                            const R* g, const F0& f0, R hMax, double* eig,
                                            R& sigmaOut) {
    constexpr int C = P::N / L;
    constexpr int kItMax = 50;
    const R kUround(2.22e-16);
    const R sqrtU = sqrt_(kUround);
    const R small = R(1.0) / hMax;
    R v[C], tmp[C];
    R nrmY(0.0), nrmV(0.0);
    {  // ||y|| and ||v|| (spectral_radius.cpp:11-13, :33-34): two chains at once
#pragma unroll
        for (int c = 0; c < C; ++c) {
            tmp[c] = y[c] * y[c];
            v[c] = R(eig[c]) * R(eig[c]);
        }
        if constexpr (is_exact<R>::value || L == 1 || BODE_RKC_SUM == 0) {
            seq_sum2<R, L, C>(G, tmp, v, nrmY, nrmV);
        } else {
            nrmY = rkc_seq_sum<R, L, C>(G, tmp, nrmY);
            nrmV = rkc_seq_sum<R, L, C>(G, v, nrmV);
        }
        nrmY = sqrt_(nrmY);
        nrmV = sqrt_(nrmV);
    }
    R dynrm;
    if (nrmY != R(0.0) && nrmV != R(0.0)) {
        dynrm = nrmY * sqrtU;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = y[c] + R(eig[c]) * (dynrm / nrmV);
    } else if (nrmY != R(0.0)) {
        dynrm = nrmY * sqrtU;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = y[c] * (R(1.0) + sqrtU);
    } else if (nrmV != R(0.0)) {
        dynrm = kUround;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = R(eig[c]) * (dynrm / nrmV);
    } else {
        dynrm = kUround;
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = kUround;
        if constexpr (is_runtime_dim<P>::value) {  // padding stays +0.0
#pragma unroll
            for (int c = 0; c < C; ++c)
                if (G.lane * C + c >= dim_of<P>(g)) v[c] = R(0.0);
        }
    }
    R sigma(0.0);
    int iters = 0;
    bool run = on;
#pragma unroll 1
    for (int iter = 1; iter <= kItMax; ++iter) {
        if constexpr (L > 1)
            if (!phase_any<L>(run)) break;
        R fv[C];
        P::template rhs<R, L>(G, t, v, g, fv);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const R d = fv[c] - f0[c];
            tmp[c] = d * d;
        }
        const R diffNrm = sqrt_(rkc_seq_sum<R, L, C>(G, tmp, R(0.0)));
        if (L == 1 || run) {  // one lane per system: always on (rkc_system_lane)
            iters = iter;
            const R sigmaOld = sigma;
            sigma = diffNrm / dynrm;
            if (iter >= 2 && fabs_(sigma - sigmaOld) <= fmax_(sigma, small) * R(0.01)) {
                if constexpr (L == 1) break;
                run = false;
            } else if (diffNrm != R(0.0)) {
#pragma unroll
                for (int c = 0; c < C; ++c) v[c] = y[c] + (fv[c] - f0[c]) * (dynrm / diffNrm);
            } else {  // degenerate direction: flip one component about y
                const int ind = iter % dim_of<P>(g);
#pragma unroll
                for (int c = 0; c < C; ++c)
                    if (G.lane * C + c == ind) v[c] = y[c] - (v[c] - y[c]);
            }
        }
    }
    sigmaOut = R(1.2) * sigma;
    if (on) {
#pragma unroll
        for (int c = 0; c < C; ++c) eig[c] = val(v[c] - y[c]);
    }
    return iters;
}

// One RKC stage j >= 2 (rkc.cpp:99-112): dst <- w_j from src = w_{j-1} and
// dst = w_{j-2} on entry (ignored when first, i.e. w_{j-2} = y).
// Groups with `act` clear evaluate the RHS with the warp and keep dst.
template <class P, class R, int L, class Y, class F0>
__device__ __forceinline__ void rkc_stage(const Group<L>& G, bool act, R tj, const Y& y,
                                          const F0& f0, const R* g,
                                          const R (&src)[P::N / L], R (&dst)[P::N / L], R muj,
                                          R nuj, R mujh, R gjh, bool first) {
    constexpr int C = P::N / L;
    R f[C];
    P::template rhs<R, L>(G, tj, src, g, f);
    if (!act) return;
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

// initialStep (rkc.cpp:146-171): one RHS at t + h on y + h f0 and the RMS
// of (f1 - f0) / (absTol + relTol |y|); wa and wb are scratch. Every lane of
// a group (of the warp, for L > 1) must call it; groups with `on` clear skip
// the scalar tail and get a meaningless value.
template <class P, class R, int L, class Y, class F0>
__device__ __forceinline__ R rkc_initial_step(const Group<L>& G, bool on, R t, const Y& ys,
                                              const F0& f0, const R* g, R wsSpecRad, R hMin,
                                              R hMax, R absTol, R relTol, R (&wa)[P::N / L],
                                              R (&wb)[P::N / L]) {
    constexpr int C = P::N / L;
    R h = hMax;
    if (wsSpecRad * h > R(1.0)) h = R(1.0) / wsSpecRad;
    h = fmax_(h, hMin);
#pragma unroll
    for (int c = 0; c < C; ++c) wa[c] = ys[c] + h * f0[c];
    P::template rhs<R, L>(G, t + h, wa, g, wb);
    elementwise_quotients<R, C, is_runtime_dim<P>::value>([&](int c) { return wb[c] - f0[c]; },
                                [&](int c) { return absTol + relTol * fabs_(ys[c]); }, wa);
#pragma unroll
    for (int c = 0; c < C; ++c) wa[c] = wa[c] * wa[c];
    const R sum = rkc_seq_sum<R, L, C>(G, wa, R(0.0));
    if (!on) return hMax;
    const R err = h * sqrt_(div_by_dim<P>(sum, g));
    if (R(0.1) * h < hMax * sqrt_(err))
        return fmax_(R(0.1) * h / sqrt_(err), hMin);
    return hMax;
}

// errorNorm (rkc.cpp:119-129) of the trial y1 = wa with f(t + h, y1) = wb.
template <class P, class R, int L, class Y, class F0>
__device__ __forceinline__ R rkc_error_norm(const Group<L>& G, const R* g, const Y& ys,
                                            const R (&y1)[P::N / L],
                                            const F0& f0, const R (&f1)[P::N / L], R h, R absTol,
                                            R relTol) {
    constexpr int C = P::N / L;
    R terms[C];
    elementwise_quotients<R, C, is_runtime_dim<P>::value>(
        [&](int c) { return R(0.8) * (ys[c] - y1[c]) + R(0.4) * h * (f0[c] + f1[c]); },
        [&](int c) { return absTol + relTol * fmax_abs(ys[c], y1[c]); }, terms);
#pragma unroll
    for (int c = 0; c < C; ++c) terms[c] = terms[c] * terms[c];
    return sqrt_(div_by_dim<P>(rkc_seq_sum<R, L, C>(G, terms, R(0.0)), g));
}

// stageCount (rkc.cpp:131-144) for the spectral radius estimate wsSpecRad
// (non-finite -> 0, rkc.cpp:240); shortens wsH when s would exceed mMax.
template <class R>
__device__ __forceinline__ long long rkc_stage_count(R wsSpecRad, long long mMax, R& wsH) {
    const R sigma = isfinite_(wsSpecRad) ? wsSpecRad : R(0.0);
    const R raw = sqrt_(R(1.54) * wsH * sigma + R(1.0));
    long long s = (raw < R(double(mMax))) ? 1 + (long long)val(raw) : mMax + 1;
    if (s > mMax) {
        s = mMax;
        wsH = (R(double(s)) * R(double(s)) - R(1.0)) / (R(1.54) * sigma);
    }
    return s;
}

// The accept/reject decision and both step-size controllers after an attempt
// (rkc.cpp:252-275, nextStepAccepted/Rejected :173-191) on the driver's
// Workspace (wsErrOld, wsHOld, wsH) plus cbErrOld = cbrt(wsErrOld). Returns
// whether the step was accepted; the caller then advances y and f0 (FSAL).
template <class R>
__device__ __forceinline__ bool rkc_finish_attempt(R err, R h, R hMin, R hMax, R uround, R cbrtU,
                                                   double p1, DevStats& st, R& t,
                                                   long long& numStep, R& wsErrOld, R& cbErrOld,
                                                   R& wsHOld, R& wsH, R& hNewRej) {
    // one cbrt call site (glibc's algorithm inline under EXACT) for both
    // controllers (rkc.cpp:177-190): cbrt(err) whenever err is finite
    const R cb = isfinite_(err) ? cbrt_(err) : R(1.0);
    if (!(err <= R(1.0))) {
        ++st.steps_rejected;
        hNewRej = isfinite_(err) ? R(0.8) * h / cb : R(p1) * h;
        return false;
    }
    t += h;
    ++numStep;
    stats_accept(st, val(h));
    const bool firstAccepted = wsHOld < uround;
    // nextStepAccepted (rkc.cpp:173-187); cbrt(errOld) is the previous
    // accepted step's cbrt(err) unless errOld was floored at uround
    R fac(10.0);
    if (firstAccepted) {
        if (R(0.8) < fac * cb) fac = R(0.8) / cb;
    } else {
        const R t1 = R(0.8) * h * cbErrOld;
        const R t2 = wsHOld * cb * cb;
        if (t1 < fac * t2) fac = t1 / t2;
    }
    const R hNew = fmax_(hMin, fmin_(hMax, h * fmax_(R(0.1), fac)));
    wsErrOld = fmax_(err, uround);
    cbErrOld = (err > uround) ? cb : cbrtU;  // errOld floored at uround
    wsHOld = h;
    wsH = hNew;
    return true;
}

// rkc::driver (rkc.cpp:193-281) with one lane per system: the same state
// machine as rkc_system below, each lane branching on its own state. (The
// warp-uniform form measured 5% slower here: with no shuffles to save, its
// extra predication only costs.)
template <class P, class R, int INSTR>
__device__ __forceinline__ void rkc_system_lane(const Group<1>& G, double t_in, double tEnd_in,
                                                R (&y)[P::N], const R* g, const DevTol& tol,
                                                DevStats& st_out) {
    constexpr int L = 1;
    constexpr int C = P::N;
    extern __shared__ double bode_smem[];
    DevStats& st = *reinterpret_cast<DevStats*>(bode_smem + threadIdx.x * kRkcSmemStride<C>() + 2 * C);
    stats_init(st);
    const R tEnd(tEnd_in);
    R t(t_in);
    const R uround(tol.uround), absTol(tol.abs_tol), relTol(tol.rel_tol), kappa(tol.kappa);
    const R hMax = fabs_(tEnd - t);
    // stageCount's mMax (rkc.cpp:132-133), a per-call constant
    long long mMax = llround(val(sqrt_(relTol / (R(10.0) * uround))));
    if (mMax < 2) mMax = 2;

    R wsErrOld(0.0), wsHOld(0.0), wsH(0.0), wsSpecRad(0.0);  // Workspace::reset
    R cbErrOld(0.0);  // cbrt(wsErrOld), valid once a step was accepted
    const R cbrtU = cbrt_(uround);  // cbrt(errOld) when errOld is floored at uround
    long long numStep = 0;
    AttemptBudget<(INSTR >= 1)> bud;
    bud.init(tol);
    // f0 and the power-method eigenvector live in this lane's shared-memory
    // row (stride kRkcSmemStride<C>, odd => conflict-free): f0 is read once
    // per element per stage, eig only by the power method; registers go to
    // y and the two stage vectors.
    double* const eig = bode_smem + threadIdx.x * kRkcSmemStride<C>();
    F0Store<R, C, kRkcF0InSmem> f0(eig + C);
    F0Store<R, C, kRkcYInSmem && (C >= 4)> ys(eig + 2 * C + 8);
    {
        R f[C];
        P::template rhs<R, L>(G, t, y, g, f);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            f0.set(c, f[c]);
            eig[c] = val(f[c]);  // rkc.cpp:212
            ys.set(c, y[c]);
        }
    }
    ++st.rhs_evals;

    int state = kTop;
    R hMin(0.0), hNewRej(0.0);
    BODE_PHASE_DECL
#pragma unroll 1
    for (;;) {
        BODE_PHASE_CTRL_END
        if (state == kTop) {
            if (!(tEnd - t > uround * fabs_(tEnd))) break;
            if (bud.spent(st)) break;
            hMin = R(10.0) * uround * fmax_(fabs_(t), hMax);
            if (R(1.1) * wsH >= fabs_(tEnd - t)) wsH = fabs_(tEnd - t);
            state = (numStep % 25 == 0) ? kSrThenAttempt : kAttempt;
        }
        BODE_PHASE_MARK(-1);
        if (state == kSrThenAttempt || state == kSrThenRejectTail) {
            R sig;
            const int it = power_method<P, R, L>(G, true, t, ys, g, f0, hMax, eig, sig);
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
        BODE_PHASE_MARK(0);
        // ---- state == kAttempt ----
        R wa[C], wb[C];
        if (wsH < uround) {  // initialStep (rkc.cpp:146-171), one RHS
            wsH = rkc_initial_step<P, R, L>(G, true, t, ys, f0, g, wsSpecRad, hMin, hMax, absTol,
                                            relTol, wa, wb);
            ++st.rhs_evals;
        }
        const long long s = rkc_stage_count(wsSpecRad, mMax, wsH);
        const R h = wsH;
        BODE_PHASE_MARK(1);
        // ---- rkc::step (rkc.cpp:82-117) with coefficients (rkc.cpp:29-69)
        // from the per-device table for s <= kRkcTableMaxS, else generated ----
        const double* crow = (tol.rkc_coef != nullptr && s <= kRkcTableMaxS)
                                 ? tol.rkc_coef + rkc_table_row(s)
                                 : nullptr;
        RkcCoefGen<R> gen;                // generator path only (local memory)
        double chunk[5 * kRkcGenChunk];  // generator path only (local memory)
        R mu1;
        if (crow != nullptr) {
            mu1 = R(crow[0]);
        } else {
            double m;
            rkc_gen_start<R>(&gen, s, val(kappa), &m);
            mu1 = R(m);
        }
        {
            const R mu1h = mu1 * h;  // muTilde_1 * h
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = ys[c] + mu1h * f0[c];
        }
        bool inA = true;  // current w_{j-1} lives in wa
        int jc = 0;       // generator path: position in the current chunk
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
                if (jc == 0)
                    rkc_gen_chunk<R>(&gen, j, j + kRkcGenChunk - 1 < s ? j + kRkcGenChunk - 1 : s,
                                     chunk);
                const double* e = chunk + 5 * jc;
                muj = R(e[0]);
                nuj = R(e[1]);
                muTj = R(e[2]);
                gTj = R(e[3]);
                cjm1 = R(e[4]);
                jc = (jc + 1 == kRkcGenChunk) ? 0 : jc + 1;
            }
            const R tj = t + cjm1 * h;
            if (inA)
                rkc_stage<P, R, L>(G, true, tj, ys, f0, g, wa, wb, muj, nuj, muTj * h, gTj * h, j == 2);
            else
                rkc_stage<P, R, L>(G, true, tj, ys, f0, g, wb, wa, muj, nuj, muTj * h, gTj * h, false);
            inA = !inA;
        }
        if (!inA) {  // y_trial = w_s -> wa
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = wb[c];
        }
        st.rhs_evals += s - 1;
        st.stages_total += s;
        BODE_PHASE_MARK(2);
        P::template rhs<R, L>(G, t + h, wa, g, wb);  // f_trial (rkc.cpp:247)
        ++st.rhs_evals;
        const R err = rkc_error_norm<P, R, L>(G, g, ys, wa, f0, wb, h, absTol, relTol);
        BODE_PHASE_MARK(3);
        BODE_PHASE_CTRL_BEGIN
        trace_step<(INSTR == 2)>(tol, G.lane == 0, t, h, (int)s, err, err <= R(1.0));
        if (rkc_finish_attempt<R>(err, h, hMin, hMax, uround, cbrtU, tol.p1, st, t, numStep,
                                  wsErrOld, cbErrOld, wsHOld, wsH, hNewRej)) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                ys.set(c, wa[c]);
                f0.set(c, wb[c]);  // FSAL swap (rkc.cpp:276)
            }
            state = kTop;
        } else {
            state = kSrThenRejectTail;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = ys[c];
    BODE_PHASE_FLUSH
    st_out = st;
}

// rkc::driver (rkc.cpp:193-281) for a lane group's system (L > 1),
// warp-uniform: every lane of the warp runs every phase that holds a shuffle
// (power method, initial step, stage loop, error norm), each group doing or
// discarding the work by its own state. Groups with `live` clear (finished,
// frozen, or past the batch's end) ride along; G carries the full warp mask.
template <class P, class R, int L, int INSTR>
__device__ __forceinline__ void rkc_system(const Group<L>& G, bool live, double t_in,
                                           double tEnd_in, R (&y)[P::N / L], const R* g,
                                           const DevTol& tol, DevStats& st_out) {
    static_assert(L > 1, "one lane per system: rkc_system_lane");
    constexpr int C = P::N / L;
    extern __shared__ double bode_smem[];
    DevStats& st = *reinterpret_cast<DevStats*>(bode_smem + threadIdx.x * kRkcSmemStride<C, L>() + 2 * C);
    stats_init(st);
    const R tEnd(tEnd_in);
    R t(t_in);
    const R uround(tol.uround), absTol(tol.abs_tol), relTol(tol.rel_tol), kappa(tol.kappa);
    const R hMax = fabs_(tEnd - t);
    // stageCount's mMax (rkc.cpp:132-133), a per-call constant
    long long mMax = llround(val(sqrt_(relTol / (R(10.0) * uround))));
    if (mMax < 2) mMax = 2;

    R wsErrOld(0.0), wsH(0.0);  // Workspace::reset
#if BODE_RKC_CTRL_SMEM
    double* const ctrl = bode_smem + threadIdx.x * kRkcSmemStride<C, L>() + kRkcCtrlOffset<C>();
    R& cbErrOld = *reinterpret_cast<R*>(ctrl);      // cbrt(wsErrOld), once a step was accepted
    R& wsHOld = *reinterpret_cast<R*>(ctrl + 1);
    R& hNewRej = *reinterpret_cast<R*>(ctrl + 2);
    R& wsSpecRad = *reinterpret_cast<R*>(ctrl + 3);
    R& cbrtU = *reinterpret_cast<R*>(ctrl + 4);     // cbrt(errOld) when errOld is floored at uround
    cbErrOld = R(0.0);
    wsHOld = R(0.0);
    hNewRej = R(0.0);
    wsSpecRad = R(0.0);
    cbrtU = cbrt_(uround);
#else
    R wsHOld(0.0), wsSpecRad(0.0), hNewRej(0.0);
    R cbErrOld(0.0);  // cbrt(wsErrOld), valid once a step was accepted
    const R cbrtU = cbrt_(uround);  // cbrt(errOld) when errOld is floored at uround
#endif
    long long numStep = 0;
    AttemptBudget<(INSTR >= 1)> bud;
    bud.init(tol);
    // f0 and the power-method eigenvector live in this lane's shared-memory
    // row (stride kRkcSmemStride<C, L>, odd => conflict-free): f0 is read once
    // per element per stage, eig only by the power method; registers go to
    // y and the two stage vectors.
    double* const eig = bode_smem + threadIdx.x * kRkcSmemStride<C, L>();
    F0Store<R, C, kRkcF0InSmem> f0(eig + C);
    F0Store<R, C, kRkcYInSmem && (C >= 4)> ys(eig + 2 * C + 8);
    {
        R f[C];
        P::template rhs<R, L>(G, t, y, g, f);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            f0.set(c, f[c]);
            eig[c] = val(f[c]);  // rkc.cpp:212
            ys.set(c, y[c]);
        }
    }
    ++st.rhs_evals;

    int state = kTop;
    R hMin(0.0);
    // The scalar transitions (no shuffles): the tail of a rejection
    // (rkc.cpp:255-264) and the top of the loop (rkc.cpp:223-229).
    auto advance = [&]() {
        if (live && state == kRejectTail) {
            if (hNewRej < hMin) {  // freeze at the last accepted state (rkc.cpp:260-263)
                st.underflow = 1;
                live = false;
            } else {
                wsH = hNewRej;
                state = kTop;
            }
        }
        if (live && state == kTop) {
            if (!(tEnd - t > uround * fabs_(tEnd))) {
                live = false;
            } else if (bud.spent(st)) {
                live = false;
            } else {
                hMin = R(10.0) * uround * fmax_(fabs_(t), hMax);
                if (R(1.1) * wsH >= fabs_(tEnd - t)) wsH = fabs_(tEnd - t);
                state = (numStep % 25 == 0) ? kSrThenAttempt : kAttempt;
            }
        }
    };
    BODE_PHASE_DECL
#pragma unroll 1
    for (;;) {
        BODE_PHASE_CTRL_END
        advance();
        if (!phase_any<L>(live)) break;
        BODE_PHASE_MARK(-1);
        const bool sr = live && (state == kSrThenAttempt || state == kSrThenRejectTail);
        if (phase_any<L>(sr)) {
            R sig;
            const int it = power_method<P, R, L>(G, sr, t, ys, g, f0, hMax, eig, sig);
            if (sr) {
                wsSpecRad = sig;
                ++st.spec_rad_evals;
                st.rhs_evals += it;
                state = (state == kSrThenAttempt) ? kAttempt : kRejectTail;
            }
            advance();  // a rejection's tail and the next top, in the same pass
        }
        BODE_PHASE_MARK(0);
        const bool att = live && state == kAttempt;
        if (!phase_any<L>(att)) continue;
        // ---- attempt (groups with att set) ----
        R wa[C], wb[C];
        const bool init = att && wsH < uround;
        if (phase_any<L>(init)) {  // initialStep (rkc.cpp:146-171), one RHS
            const R h0 = rkc_initial_step<P, R, L>(G, init, t, ys, f0, g, wsSpecRad, hMin, hMax,
                                                   absTol, relTol, wa, wb);
            if (init) {
                ++st.rhs_evals;
                wsH = h0;
            }
        }
        // s = 1 (no stages) for idle groups
        const long long s = att ? rkc_stage_count(wsSpecRad, mMax, wsH) : 1;
        const R h = wsH;
        BODE_PHASE_MARK(1);
        // ---- rkc::step (rkc.cpp:82-117) with coefficients (rkc.cpp:29-69)
        // from the per-device table for s <= kRkcTableMaxS, else generated ----
        const double* crow = (att && tol.rkc_coef != nullptr && s <= kRkcTableMaxS)
                                 ? tol.rkc_coef + rkc_table_row(s)
                                 : nullptr;
        RkcCoefGen<R> gen;                // generator path only (local memory)
        double chunk[5 * kRkcGenChunk];  // generator path only (local memory)
        R mu1(0.0);
        if (att) {
            if (crow != nullptr) {
                mu1 = R(crow[0]);
            } else {
                double m;
                rkc_gen_start<R>(&gen, s, val(kappa), &m);
                mu1 = R(m);
            }
        }
        {
            const R mu1h = mu1 * h;  // muTilde_1 * h
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = ys[c] + mu1h * f0[c];
        }
        // the warp runs max(s) - 1 stages; w_j alternates between wa and wb
        const long long sMax = (long long)__reduce_max_sync(0xffffffffu, (unsigned)s);
        bool inA = true;  // current w_{j-1} lives in wa
        int jc = 0;       // generator path: position in the current chunk
#pragma unroll 1
        for (long long j = 2; j <= sMax; ++j) {
            const bool act = j <= s;
            R muj(0.0), nuj(0.0), muTj(0.0), gTj(0.0), cjm1(0.0);
            if (act) {
                if (crow != nullptr) {  // the device table: read-only global loads
                    const double* e = crow + 1 + 5 * (j - 2);
                    muj = R(__ldg(e));
                    nuj = R(__ldg(e + 1));
                    muTj = R(__ldg(e + 2));
                    gTj = R(__ldg(e + 3));
                    cjm1 = R(__ldg(e + 4));
                } else {  // the generator's chunk in local memory
                    if (jc == 0)
                        rkc_gen_chunk<R>(&gen, j,
                                         j + kRkcGenChunk - 1 < s ? j + kRkcGenChunk - 1 : s,
                                         chunk);
                    const double* e = chunk + 5 * jc;
                    muj = R(e[0]);
                    nuj = R(e[1]);
                    muTj = R(e[2]);
                    gTj = R(e[3]);
                    cjm1 = R(e[4]);
                    jc = (jc + 1 == kRkcGenChunk) ? 0 : jc + 1;
                }
            }
            const R tj = t + cjm1 * h;
            if (inA)
                rkc_stage<P, R, L>(G, act, tj, ys, f0, g, wa, wb, muj, nuj, muTj * h, gTj * h,
                                   j == 2);
            else
                rkc_stage<P, R, L>(G, act, tj, ys, f0, g, wb, wa, muj, nuj, muTj * h, gTj * h,
                                   false);
            inA = !inA;
        }
        if ((s & 1) == 0) {  // the last stage (j = s even) wrote wb: y_trial -> wa
#pragma unroll
            for (int c = 0; c < C; ++c) wa[c] = wb[c];
        }
        BODE_PHASE_MARK(2);
        P::template rhs<R, L>(G, t + h, wa, g, wb);  // f_trial (rkc.cpp:247)
        const R err = rkc_error_norm<P, R, L>(G, g, ys, wa, f0, wb, h, absTol, relTol);
        BODE_PHASE_MARK(3);
        BODE_PHASE_CTRL_BEGIN
        if (!att) continue;
        st.rhs_evals += s;  // s - 1 stages and f_trial
        st.stages_total += s;
        trace_step<(INSTR == 2)>(tol, G.lane == 0, t, h, (int)s, err, err <= R(1.0));
        if (rkc_finish_attempt<R>(err, h, hMin, hMax, uround, cbrtU, tol.p1, st, t, numStep,
                                  wsErrOld, cbErrOld, wsHOld, wsH, hNewRej)) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                ys.set(c, wa[c]);
                f0.set(c, wb[c]);  // FSAL swap (rkc.cpp:276)
            }
            state = kTop;
        } else {
            state = kSrThenRejectTail;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = ys[c];
    BODE_PHASE_FLUSH
    st_out = st;
}

}  // namespace bode
