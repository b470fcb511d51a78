// rkck_pleiades2.cuh -- RKCK on the Pleiades problem with each system split
// across a pair of lanes by axis: lane 0 owns (x_1..x_7, x'_1..x'_7), lane 1
// owns (y_1..y_7, y'_1..y'_7).
//
// Same arithmetic as rkck_nystrom.cuh (and so as rkck.cpp:34-159 with
// problems.cpp:13-35): the Nystrom storage (f0 = (v, A0), k_j = (V_j, A_j))
// and the step/error/controller sequence are unchanged; only the work is
// distributed:
//   * stage arguments, V_j, yNext and the error-norm terms are per component,
//     so each lane does its own axis;
//   * the acceleration needs every position: the lanes swap their 7
//     positions (shuffles), each computes 1/r^3 for half of the 21 pairs
//     (interleaved by pair index) and the halves are swapped back;
//   * each lane then accumulates its own axis over all 21 pairs in the
//     reference's (i outer, j inner) order -- the x and y accumulators never
//     mix in the reference either, so every sum is bitwise the reference's;
//   * r2 = dx*dx + dy*dy is computed by the lane that owns the pair; IEEE
//     addition is commutative, so (own^2 + other^2) is the reference value;
//   * the error norm's max is combined across the pair (order-independent),
//     and both lanes then run the identical scalar controller.
// Per lane: 21 doubles of state in registers and 4 stage slots of 14 doubles
// in shared memory (456 B), which lets ~12 warps share an SM instead of 8.
#pragma once

#include "rkck_nystrom.cuh"

namespace bode {

// pair p = (i, j), i < j, in the reference's loop order
__host__ __device__ constexpr int pl_pair_i(int p) {
    return p < 6 ? 0 : p < 11 ? 1 : p < 15 ? 2 : p < 18 ? 3 : p < 20 ? 4 : 5;
}
__host__ __device__ constexpr int pl_pair_j(int p) {
    return p < 6 ? p + 1 : p < 11 ? p - 4 : p < 15 ? p - 8 : p < 18 ? p - 11 : p < 20 ? p - 13 : 6;
}

// Accelerations of this lane's axis; Q = own-axis positions. Each lane squares
// its axis' differences for all 21 pairs and swaps them with its partner, so
// both know r2 = dx*dx + dy*dy (IEEE addition commutes: bitwise the
// reference's); lane l then evaluates 1/(r2 sqrt r2) for pairs p = 2k + l and
// the two halves are swapped back. The instruction stream is lane-uniform.
template <class R>
__device__ __forceinline__ void pleiades_accel_pair(const Group<2>& G, const R* Q, R (&a)[7]) {
    double sq[21];
#pragma unroll
    for (int p = 0; p < 21; ++p) {
        const R d = Q[pl_pair_j(p)] - Q[pl_pair_i(p)];
        sq[p] = val(d * d);
    }
    double mine[11], r2s[11];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        const int p0 = 2 * k, p1 = (2 * k + 1 < 21) ? 2 * k + 1 : 20;
        const double s0 = __shfl_xor_sync(0xffffffffu, sq[p0], 1);
        const double s1 = __shfl_xor_sync(0xffffffffu, sq[p1], 1);
        // lane 0 takes pair p0, lane 1 pair p1 (lane 1 repeats pair 20 at k = 10)
        const double own = G.lane ? sq[p1] : sq[p0];
        const double oth = G.lane ? s1 : s0;
        if constexpr (is_exact<R>::value) {  // straight-line IEEE ops (arith.cuh)
            const double r2 = __dadd_rn(own, oth);
            const double d = __dmul_rn(r2, sqrt_rn_bf(r2));
            ok = ok & r3_in_safe_range(r2);
            r2s[k] = r2;
            mine[k] = rcp_rn_bf(d);
        } else {
            mine[k] = rsqrt3_fast(own + oth);
        }
    }
    if constexpr (is_exact<R>::value) {
        if (!ok) {  // rare: an operand outside [2^-400, 2^400] (or NaN/Inf)
#pragma unroll
            for (int k = 0; k < 11; ++k)
                mine[k] = __ddiv_rn(1.0, __dmul_rn(r2s[k], __dsqrt_rn(r2s[k])));
        }
    }
    double other[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) other[k] = __shfl_xor_sync(0xffffffffu, mine[k], 1);
#pragma unroll
    for (int i = 0; i < 7; ++i) a[i] = R(0.0);
#pragma unroll
    for (int p = 0; p < 21; ++p) {
        const int i = pl_pair_i(p), j = pl_pair_j(p);
        // pair p was evaluated by lane p & 1 in its round p >> 1
        const double inv = ((p & 1) == G.lane) ? mine[p >> 1] : other[p >> 1];
        const R d = Q[j] - Q[i];
        const double mi = double(i + 1), mj = double(j + 1);
        if constexpr (is_exact<R>::value) {
            a[i] += R(mj) * d * R(inv);
            a[j] -= R(mi) * d * R(inv);
        } else {
            const double t = val(d) * inv;
            a[i] += mj * t;
            a[j] -= mi * t;
        }
    }
}

template <class R, int INSTR>
__device__ __forceinline__ void rkck_pleiades2_system(const Group<2>& G, double t_in,
                                                      double tEnd_in, R (&y)[14],
                                                      const DevTol& tol, DevStats& st) {
    constexpr int M = 7;   // components per half (positions or velocities of one axis)
    constexpr int W = 14;  // doubles per stage slot per lane
    using namespace ck;
    stats_init(st);
    extern __shared__ double bode_smem[];
    double* const ks = bode_smem + threadIdx.x * kSmemStride<14>();
    auto kget = [&](int m, int c) -> R { return R(ks[m * W + c]); };
    auto kset = [&](int m, int c, R v) { ks[m * W + c] = val(v); };

    R* const q = y;      // own-axis positions
    R* const v = y + M;  // own-axis velocities
    const R tEnd(tEnd_in);
    R t(t_in);
    const R hMax = fabs_(tEnd - t);
    const R hMin(tol.h_min_floor);
    R h = R(0.5) * fabs_(tEnd - t);
    const R uround(tol.uround), eps(tol.eps), tiny(tol.tiny);

    R A0[M];
    bool haveF = false;
    bool live = tEnd - t > uround * fabs_(tEnd);  // rkck.cpp:131
    AttemptBudget<(INSTR >= 1)> bud;
    bud.init(tol);

    // Warp-uniform loop: the warp iterates while any of its systems is live,
    // so every shuffle runs with the full mask (no collective fix-up code).
    // Finished systems ride along with their state and stats frozen -- the
    // SIMT cost is the same as the divergent loop's masked iterations.
#pragma unroll 1
    while (__any_sync(0xffffffffu, live)) {
        if (live) h = fmin_(tEnd - t, h);
        // One call site for the pair RHS: j = 1 is f(t, y) when any lane
        // needs it (rkck.cpp:133-137), j = 2..6 the stages (rkck.cpp:42-64).
        // A single inlined copy keeps the kernel small enough for the
        // instruction cache.
        R Q[M], Acc[M];
#pragma unroll 1
        for (int j = __any_sync(0xffffffffu, live && !haveF) ? 1 : 2; j <= 6; ++j) {
            const int out = (j == 6) ? 0 : j - 2;  // k6 reuses k2's slot
            if (j == 1) {
#pragma unroll
                for (int i = 0; i < M; ++i) Q[i] = q[i];
            } else if (j == 2) {  // stage 2: y + h*b21*f0
                const R hb = h * R(b21);
#pragma unroll
                for (int i = 0; i < M; ++i) kset(0, i, v[i] + hb * A0[i]);
#pragma unroll
                for (int i = 0; i < M; ++i) Q[i] = q[i] + hb * v[i];
            } else {
                const double b0 = c_ck_b[j - 3][0];
                double bm[4];  // b_j2..b_j5 (zero past the stage's last term)
#pragma unroll
                for (int m = 0; m < 4; ++m) bm[m] = c_ck_b[j - 3][m + 1];
                const int nk = j - 2;
                // the newest acceleration A_{j-1} is still in Acc; it is the last
                // term of every stage sum, so reading it from registers keeps the
                // reference's summation order
                const double blast = c_ck_b[j - 3][nk];
                if constexpr (is_exact<R>::value) {
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        R s = R(b0) * A0[i];
#pragma unroll
                        for (int m = 0; m < 3; ++m)  // predicated: constant offsets, no loop
                            if (m < nk - 1) s = s + R(bm[m]) * kget(m, M + i);
                        s = s + R(blast) * Acc[i];
                        Acc[i] = v[i] + h * s;
                    }
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        R s = R(b0) * v[i];
#pragma unroll
                        for (int m = 0; m < 4; ++m)
                            if (m < nk) s = s + R(bm[m]) * kget(m, i);
                        Q[i] = q[i] + h * s;
                    }
                } else {  // FAST: h folded into the stage weights (rkck_nystrom.cuh)
                    const double hb0 = val(h) * b0;
                    double hbm[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) hbm[m] = val(h) * bm[m];
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        double s = fma(hb0, val(A0[i]), val(v[i]));
#pragma unroll
                        for (int m = 0; m < 3; ++m)
                            if (m < nk - 1) s = fma(hbm[m], val(kget(m, M + i)), s);
                        Acc[i] = R(fma(val(h) * blast, val(Acc[i]), s));
                    }
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        double s = fma(hb0, val(v[i]), val(q[i]));
#pragma unroll
                        for (int m = 0; m < 4; ++m)
                            if (m < nk) s = fma(hbm[m], val(kget(m, i)), s);
                        Q[i] = R(s);
                    }
                }
#pragma unroll
                for (int i = 0; i < M; ++i) kset(out, i, Acc[i]);
            }
            pleiades_accel_pair<R>(G, Q, Acc);
            if (j == 1) {
                if (live && !haveF) {
#pragma unroll
                    for (int i = 0; i < M; ++i) A0[i] = Acc[i];
                    ++st.rhs_evals;
                    haveF = true;
                }
            } else if (j != 6) {  // A6 stays in Acc for the error norm and yNext
#pragma unroll
                for (int i = 0; i < M; ++i) kset(out, M + i, Acc[i]);
            }
        }
        if (live) {
            st.rhs_evals += 5;
            st.stages_total += 6;
        }

        // error norm (rkck.cpp:75-76, :88-98), own components, then across the pair
        R err;
        bool nanFlag = false;
        {
            // four interleaved accumulators: max and exact-argmax are associative,
            // so this only shortens the dependency chain (4x), never the result
            // the max is tracked as an exact (EXACT) or rounded (FAST) argmax by
            // cross-multiplication and divided out once (arith.cuh QuotMax)
            QuotMax qm[4];
            double ma[4] = {0.0, 0.0, 0.0, 0.0}, mb[4] = {1.0, 1.0, 1.0, 1.0};
            const double hh = val(h);
            const double hd1 = hh * d1, hd3 = hh * d3, hd4 = hh * d4, hd5 = hh * d5, hd6 = hh * d6;
            int bad = 0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const R k0q = kget(0, i), k1q = kget(1, i), k2q = kget(2, i);
                const R k0v = Acc[i], k1v = kget(1, M + i), k2v = kget(2, M + i);  // A6 = Acc
                if constexpr (is_exact<R>::value) {
                    const R eq = h * (R(d1) * v[i] + R(d3) * k1q + R(d4) * k2q +
                                      R(d5) * kget(3, i) + R(d6) * k0q);
                    const R ev = h * (R(d1) * A0[i] + R(d3) * k1v + R(d4) * k2v +
                                      R(d5) * kget(3, M + i) + R(d6) * k0v);
                    // candidate yNext (rkck.cpp:74), kept only if the step is accepted
                    Q[i] = q[i] + h * (R(c1) * v[i] + R(c3) * k1q + R(c4) * k2q + R(c6) * k0q);
                    Acc[i] = v[i] + h * (R(c1) * A0[i] + R(c3) * k1v + R(c4) * k2v + R(c6) * k0v);
                    if (!isfinite_(eq) || !isfinite_(ev)) nanFlag = true;
                    const R dq = fabs_(q[i]) + fabs_(h * v[i]) + tiny;
                    const R dv = fabs_(v[i]) + fabs_(h * A0[i]) + tiny;
                    qm[(2 * i) & 3].push(fabs(val(eq)), val(dq));
                    qm[(2 * i + 1) & 3].push(fabs(val(ev)), val(dv));
                } else {
                    const double eq = fma(hd6, val(k0q), fma(hd5, val(kget(3, i)),
                                      fma(hd4, val(k2q), fma(hd3, val(k1q), hd1 * val(v[i])))));
                    const double ev = fma(hd6, val(k0v), fma(hd5, val(kget(3, M + i)),
                                      fma(hd4, val(k2v), fma(hd3, val(k1v), hd1 * val(A0[i])))));
                    Q[i] = R(fma(hh * c6, val(k0q), fma(hh * c4, val(k2q),
                             fma(hh * c3, val(k1q), fma(hh * c1, val(v[i]), val(q[i]))))));
                    Acc[i] = R(fma(hh * c6, val(k0v), fma(hh * c4, val(k2v),
                               fma(hh * c3, val(k1v), fma(hh * c1, val(A0[i]), val(v[i]))))));
                    bad |= ((__double2hiint(eq) & 0x7ff00000) == 0x7ff00000) |
                           ((__double2hiint(ev) & 0x7ff00000) == 0x7ff00000);
                    const double dq = fma(hh, fabs(val(v[i])), fabs(val(q[i]))) + val(tiny);
                    const double dv = fma(hh, fabs(val(A0[i])), fabs(val(v[i]))) + val(tiny);
                    const int kq = (2 * i) & 3, kv = (2 * i + 1) & 3;
                    if (fabs(eq) * mb[kq] > ma[kq] * dq) { ma[kq] = fabs(eq); mb[kq] = dq; }
                    if (fabs(ev) * mb[kv] > ma[kv] * dv) { ma[kv] = fabs(ev); mb[kv] = dv; }
                }
            }
            if constexpr (is_exact<R>::value) {
                qm[0].push(qm[1].a, qm[1].b);
                qm[2].push(qm[3].a, qm[3].b);
                qm[0].push(qm[2].a, qm[2].b);
                nanFlag = (__ballot_sync(0xffffffffu, nanFlag) & G.mask) != 0u;
                qm[0].push(__shfl_xor_sync(0xffffffffu, qm[0].a, 1),
                           __shfl_xor_sync(0xffffffffu, qm[0].b, 1));
                err = R(qm[0].value()) / eps;
            } else {
#pragma unroll
                for (int k = 1; k < 4; ++k)
                    if (ma[k] * mb[0] > ma[0] * mb[k]) { ma[0] = ma[k]; mb[0] = mb[k]; }
                nanFlag = (__ballot_sync(0xffffffffu, bad != 0) & G.mask) != 0u;
                const double oa = __shfl_xor_sync(0xffffffffu, ma[0], 1);
                const double ob = __shfl_xor_sync(0xffffffffu, mb[0], 1);
                if (oa * mb[0] > ma[0] * ob) { ma[0] = oa; mb[0] = ob; }
                err = R(ma[0] * rcp_fast(mb[0] * val(eps)));
            }
        }

        R hNew;
        bool accepted;
        if constexpr (is_exact<R>::value) {
            accepted = rkck_adjust(h, err, nanFlag, hMin, hMax, tol, hNew);
        } else {
            if (err > 1.0 || !isfinite(err) || nanFlag) {
                accepted = false;
                hNew = (!isfinite(err) || nanFlag)
                           ? tol.p1 * h
                           : fmax(tol.safety * h * ctrl_pow_fast(err, tol.pshrnk), tol.p1 * h);
            } else {
                accepted = true;
                const double hn =
                    (err > tol.errcon) ? tol.safety * h * ctrl_pow_fast(err, tol.pgrow) : 5.0 * h;
                hNew = fmax(val(hMin), fmin(val(hMax), hn));
            }
        }
        trace_step<(INSTR == 2)>(tol, live && G.lane == 0, t, h, 6, err, accepted);
        if (live && accepted) {
            t += h;
            stats_accept(st, val(h));
            // yNext (rkck.cpp:74), formed with the error norm
#pragma unroll
            for (int i = 0; i < M; ++i) {
                q[i] = Q[i];
                v[i] = Acc[i];
            }
            haveF = false;
            h = hNew;
        } else if (live) {
            ++st.steps_rejected;
            if (hNew < R(tol.h_min_floor)) {  // freeze at the last accepted state
                st.underflow = 1;
                live = false;
            }
            h = hNew;
        }
        if (live) live = tEnd - t > uround * fabs_(tEnd);
        if (live && bud.spent_after(st)) live = false;
    }
}

}  // namespace bode
