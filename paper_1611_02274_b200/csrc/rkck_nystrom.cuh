// rkck_nystrom.cuh -- RKCK for second-order systems y = (q, v), dq/dt = v,
// dv/dt = a(q) (the Pleiades problem, problems.cpp:13-35).
//
// This is rkck::step / errorNorm / adjustStep / driver (rkck.cpp:34-159)
// evaluated on the same operands in the same order, but stored in Nystrom
// form: for such an RHS the first half of every stage derivative is a copy
// of the second half of its stage argument (problems.cpp:17,
// out[i] = w[14 + i]), so
//   f0      = (v, A0)            -- only A0 = a(q) is stored, v aliases y
//   k_j     = (V_j, A_j)         -- V_j = v + h * sum_m b_jm A_m
//   arg_j   = (Q_j, V_j)         -- Q_j = q + h * sum_m b_jm V_m  (V_1 = v)
// Every double that enters an operation is bitwise the one the reference
// uses, so with R = xd the result is bitwise rkck::driver's (up to the
// device pow in the controller, see arith.cuh).
//
// Register/shared-memory plan (one system per thread, SURVEY.md 7.4 hard
// part 1): q, v, A0 in registers (3 x M doubles); k2..k5 in shared memory,
// one odd-length row per thread (conflict-free, immediate offsets); stages
// 3..6 run as one rolled loop (one inlined acceleration, bounded live ranges);
// k6 reuses k2's slot (c2 = c*2 = 0, so k2 is dead once arg6 is formed); the
// error norm is folded into the step and costs one division (arith.cuh
// QuotMax); the fast policy is free of out-of-line calls.
#pragma once

#include "rkck.cuh"

namespace bode {

// Problems that declare `static constexpr bool second_order = true` and an
// accel(t, q, g, a) (problems.cuh SecondOrderProblem) take the Nystrom kernels.
template <class P, class = void>
struct is_second_order {
    static constexpr bool value = false;
};
template <class P>
struct is_second_order<P, decltype((void)P::second_order)> {
    static constexpr bool value = P::second_order;
};
template <class P>
constexpr bool is_pleiades = false;
template <>
constexpr bool is_pleiades<Pleiades> = true;
// stage nodes a3..a6 (rkck.cpp:9), for the rolled stage loop
__constant__ double c_ck_a[4] = {3.0 / 10.0, 3.0 / 5.0, 1.0, 7.0 / 8.0};

#define BODE_FENCE() asm volatile("" ::: "memory")

// b_j1..b_j5 for stages 3..6 (rkck.cpp:15-19), read uniformly by the warp
__constant__ double c_ck_b[4][5] = {
    {3.0 / 40.0, 9.0 / 40.0, 0.0, 0.0, 0.0},
    {3.0 / 10.0, -9.0 / 10.0, 6.0 / 5.0, 0.0, 0.0},
    {-11.0 / 54.0, 5.0 / 2.0, -70.0 / 27.0, 35.0 / 27.0, 0.0},
    {1631.0 / 55296.0, 175.0 / 512.0, 575.0 / 13824.0, 44275.0 / 110592.0, 253.0 / 4096.0}};

// ---- FAST policy: the same Cash-Karp step in Runge-Kutta-Nystrom form ----
// With k_m = (V_m, A_m), V_1 = v and V_m = v + h sum_l b_ml A_l, every
// position-half quantity of the step is a combination of accelerations only:
//   Q_j        = q + h a_j v + h^2 sum_{l<=j-2} BB_jl A_l,  BB_jl = sum_m b_jm b_ml
//   yNext_q    = q + h v     + h^2 sum_l CB_l A_l,          CB_l  = sum_m c_m b_ml
//   yErr_q     =               h^2 sum_l DB_l A_l,          DB_l  = sum_m d_m b_ml
// (row sums of b are the nodes a_j, sum c_m = 1, sum d_m = 0). Exact algebra,
// so the FAST step differs from the reference only by rounding, while the
// velocity stage values V_j are never formed or stored: half the stage
// storage (A_2..A_5 only), about 40% fewer stage FMAs and shared-memory
// accesses. EXACT keeps the reference's own operation sequence.
namespace rkn {
using namespace ck;
constexpr double BB[5][4] = {  // rows j = 2..6, columns l = 1..4
    {0.0, 0.0, 0.0, 0.0},
    {b32 * b21, 0.0, 0.0, 0.0},
    {b42 * b21 + b43 * b31, b43 * b32, 0.0, 0.0},
    {b52 * b21 + b53 * b31 + b54 * b41, b53 * b32 + b54 * b42, b54 * b43, 0.0},
    {b62 * b21 + b63 * b31 + b64 * b41 + b65 * b51, b63 * b32 + b64 * b42 + b65 * b52,
     b64 * b43 + b65 * b53, b65 * b54}};
constexpr double CB0 = c3 * b31 + c4 * b41 + c6 * b61, CB1 = c3 * b32 + c4 * b42 + c6 * b62,
                 CB2 = c4 * b43 + c6 * b63, CB3 = c6 * b64, CB4 = c6 * b65;
constexpr double DB0 = d3 * b31 + d4 * b41 + d5 * b51 + d6 * b61,
                 DB1 = d3 * b32 + d4 * b42 + d5 * b52 + d6 * b62,
                 DB2 = d4 * b43 + d5 * b53 + d6 * b63, DB3 = d5 * b54 + d6 * b64, DB4 = d6 * b65;
constexpr double NODE[5] = {a2, a3, a4, a5, a6};
}  // namespace rkn
__constant__ double c_rkn_bb[4][4] = {  // stages 3..6 (rolled loop)
    {rkn::BB[1][0], 0.0, 0.0, 0.0},
    {rkn::BB[2][0], rkn::BB[2][1], 0.0, 0.0},
    {rkn::BB[3][0], rkn::BB[3][1], rkn::BB[3][2], 0.0},
    {rkn::BB[4][0], rkn::BB[4][1], rkn::BB[4][2], rkn::BB[4][3]}};
__constant__ double c_rkn_node[4] = {rkn::NODE[1], rkn::NODE[2], rkn::NODE[3], rkn::NODE[4]};

// Doubles per thread in the stage-slot row: EXACT stores k2..k5 whole (4N),
// FAST (Nystrom form) only A_2..A_5 (4 N/2); odd => conflict-free.
template <class P, class R>
__host__ __device__ constexpr int nystrom_smem_doubles() {
    return is_exact<R>::value ? kSmemStride<P::N>() : kSmemStride<P::N / 2>();
}

// Per-lane solver state: one system, advanced one attempt at a time, so a
// persistent kernel can hand a lane a new system as soon as its own finishes.
constexpr bool kRkckUnrollStages = false;  // measured: unrolling adds spills, -16%

template <class P, class R, int INSTR>
struct NystromRkck {
    static constexpr int M = P::N / 2;
    R y[P::N];  // (q, v)
    R A0[M];    // acceleration half of f0 = f(t, y)
    R t, tEnd, hMax, h;
    bool haveF, live;
    DevStats st;
    AttemptBudget<(INSTR >= 1)> bud;  // bode_set_attempt_budget (off by default)
    double* ks;         // this lane's shared-memory row (k2..k5 / k6)
    const R* gp = nullptr;  // the system's parameters (problems with P > 0)

    __device__ __forceinline__ const double* gpd() const {  // params as doubles (FAST form)
        return reinterpret_cast<const double*>(gp);
    }
    __device__ __forceinline__ R kget(int m, int c) const { return R(ks[m * P::N + c]); }
    __device__ __forceinline__ void kset(int m, int c, R v) { ks[m * P::N + c] = val(v); }

    // rkck::driver prologue (rkck.cpp:119-128); y must already hold the state
    __device__ __forceinline__ void start(double t_in, double tEnd_in, const DevTol& tol) {
        extern __shared__ double bode_smem[];
        ks = bode_smem + threadIdx.x * nystrom_smem_doubles<P, R>();
        stats_init(st);
        tEnd = R(tEnd_in);
        t = R(t_in);
        hMax = fabs_(tEnd - t);
        h = R(0.5) * fabs_(tEnd - t);
        haveF = false;
        live = tEnd - t > R(tol.uround) * fabs_(tEnd);  // rkck.cpp:131
        bud.init(tol);
    }

    // one pass of the while loop of rkck.cpp:131-157
    __device__ __forceinline__ void attempt(const DevTol& tol) {
        using namespace ck;
        R* const q = y;
        R* const v = y + M;
        const R hMin(tol.h_min_floor);
        const R uround(tol.uround), eps(tol.eps), tiny(tol.tiny);
        h = fmin_(tEnd - t, h);
        if (!haveF) {  // rejected retries reuse f(t, y) (rkck.cpp:133-137)
            P::template accel<R>(t, q, gp, A0);
            ++st.rhs_evals;
            haveF = true;
        }
        if constexpr (!is_exact<R>::value) {
            attempt_rkn(tol);
            return;
        }
        R Q[M], Acc[M];
        {  // stage 2: arg = y + h*b21*f0 (rkck.cpp:42-44)
            const R hb = h * R(b21);
#pragma unroll
            for (int i = 0; i < M; ++i) kset(0, i, v[i] + hb * A0[i]);
#pragma unroll
            for (int i = 0; i < M; ++i) Q[i] = q[i] + hb * v[i];
            BODE_FENCE();
            P::template accel<R>(t + R(a2) * h, Q, gp, Acc);
#pragma unroll
            for (int i = 0; i < M; ++i) kset(0, M + i, Acc[i]);
            BODE_FENCE();
        }
        // stages 3..6 (rkck.cpp:46-64): arg = y + h*(b_j1 f0 + b_j2 k2 + ...).
        // kRkckUnrollStages: unrolled, every sum has its exact length; else one
        // rolled loop whose sums are predicated to the stage's length.
#pragma unroll
        for (int j = 3; j <= (kRkckUnrollStages ? 6 : 3); ++j) stage_block<kRkckUnrollStages>(j, Q, Acc);
#pragma unroll 1
        for (int j = 4; j <= (kRkckUnrollStages ? 3 : 6); ++j) stage_block<false>(j, Q, Acc);
        st.rhs_evals += 5;
        st.stages_total += 6;
        finish_attempt(tol, Q, Acc);
    }

    // stage j in 3..6; UNROLLED: j is a compile-time constant after unrolling
    template <bool UNROLLED>
    __device__ __forceinline__ void stage_block(int j, R (&Q)[M], R (&Acc)[M]) {
        R* const q = y;
        R* const v = y + M;
        {
            const double b0 = c_ck_b[j - 3][0];
            double bm[4];  // b_j2..b_j5 (zero past the stage's last term)
#pragma unroll
            for (int m = 0; m < 4; ++m) bm[m] = c_ck_b[j - 3][m + 1];
            const int nk = j - 2;                  // k2..k_{j-1} enter this stage
            const int out = (j == 6) ? 0 : j - 2;  // k6 reuses k2's slot
            if constexpr (is_exact<R>::value) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    R s = R(b0) * A0[i];
#pragma unroll
                    for (int m = 0; m < 4; ++m)  // predicated: constant offsets, no loop
                        if (m < nk) s = s + R(bm[m]) * kget(m, M + i);
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
            } else {  // FAST: h folded into the stage weights, one FMA per term;
                      // the newest acceleration A_{j-1} is still in Acc (no reload)
                const double hb0 = val(h) * b0;
                const double hlast = val(h) * c_ck_b[j - 3][nk];
                double hbm[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) hbm[m] = val(h) * bm[m];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    double s = fma(hb0, val(A0[i]), val(v[i]));
#pragma unroll
                    for (int m = 0; m < 3; ++m)
                        if (m < nk - 1) s = fma(hbm[m], val(kget(m, M + i)), s);
                    Acc[i] = R(fma(hlast, val(Acc[i]), s));
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
            BODE_FENCE();
#pragma unroll
            for (int i = 0; i < M; ++i) kset(out, i, Acc[i]);
            BODE_FENCE();
            P::template accel<R>(t + R(c_ck_a[j - 3]) * h, Q, gp, Acc);
            // FAST reads A6 from registers (finish_attempt), so its slot is never stored
            if (is_exact<R>::value || j != 6) {
#pragma unroll
                for (int i = 0; i < M; ++i) kset(out, M + i, Acc[i]);
            }
            BODE_FENCE();
        }
    }

    // FAST: one attempt in Nystrom form (see namespace rkn). Slots 0..3 of the
    // row hold A_2..A_5 (M doubles each); A_1 = A0 and the newest acceleration
    // stay in registers.
    __device__ __forceinline__ void attempt_rkn(const DevTol& tol) {
        using namespace ck;
        double* const q = reinterpret_cast<double*>(y);
        double* const v = reinterpret_cast<double*>(y) + M;
        const double hh = val(h), h2 = hh * hh;
        double Q[M], Acc[M];
        {  // stage 2
            const double ha = hh * a2;  // Q_2 = q + h b21 v (b21 = a2)
#pragma unroll
            for (int i = 0; i < M; ++i) Q[i] = fma(ha, v[i], q[i]);
            P::template accel<double>(val(t) + ha, Q, gpd(), Acc);
        }
        // stages 3..6: store the newest acceleration A_{j-1} (slot j-3), then
        // form Q_j from A_1..A_{j-2}
#pragma unroll 1
        for (int j = 3; j <= 6; ++j) {  // rolled: fully unrolled measured 13% slower
#pragma unroll
            for (int i = 0; i < M; ++i) ks[(j - 3) * M + i] = Acc[i];
            const double ha = hh * c_rkn_node[j - 3];
            double hb[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) hb[l] = h2 * c_rkn_bb[j - 3][l];
            BODE_FENCE();
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double s = fma(hb[0], val(A0[i]), fma(ha, v[i], q[i]));
#pragma unroll
                for (int l = 1; l < 4; ++l)  // A_{l+1} from slot l-1, predicated to l <= j-3
                    if (l <= j - 3) s = fma(hb[l], ks[(l - 1) * M + i], s);
                Q[i] = s;
            }
            P::template accel<double>(val(t) + ha, Q, gpd(), Acc);
        }
        st.rhs_evals += 5;
        st.stages_total += 6;
        // error norm (rkck.cpp:75-76, :88-98) and the candidate yNext in one
        // pass over A_2..A_5; A6 = Acc
        const double eps = tol.eps, tiny = tol.tiny;
        const double hd1 = hh * d1, hd3 = hh * d3, hd4 = hh * d4, hd5 = hh * d5, hd6 = hh * d6;
        const double hc1 = hh * c1, hc3 = hh * c3, hc4 = hh * c4, hc6 = hh * c6;
        const double e2[5] = {h2 * rkn::DB0, h2 * rkn::DB1, h2 * rkn::DB2, h2 * rkn::DB3,
                              h2 * rkn::DB4};
        const double c2[5] = {h2 * rkn::CB0, h2 * rkn::CB1, h2 * rkn::CB2, h2 * rkn::CB3,
                              h2 * rkn::CB4};
        double ma[4] = {0.0, 0.0, 0.0, 0.0}, mb[4] = {1.0, 1.0, 1.0, 1.0};
        int bad = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double a1 = val(A0[i]), a2v = ks[i], a3v = ks[M + i], a4v = ks[2 * M + i],
                         a5v = ks[3 * M + i], a6v = Acc[i];
            const double eq = fma(e2[4], a5v, fma(e2[3], a4v, fma(e2[2], a3v,
                              fma(e2[1], a2v, e2[0] * a1))));
            const double ev = fma(hd6, a6v, fma(hd5, a5v, fma(hd4, a4v, fma(hd3, a3v, hd1 * a1))));
            Q[i] = fma(c2[4], a5v, fma(c2[3], a4v, fma(c2[2], a3v, fma(c2[1], a2v,
                   fma(c2[0], a1, fma(hh, v[i], q[i]))))));
            Acc[i] = fma(hc6, a6v, fma(hc4, a4v, fma(hc3, a3v, fma(hc1, a1, v[i]))));
            bad |= ((__double2hiint(eq) & 0x7ff00000) == 0x7ff00000) |
                   ((__double2hiint(ev) & 0x7ff00000) == 0x7ff00000);
            const double dq = fma(hh, fabs(v[i]), fabs(q[i])) + tiny;
            const double dv = fma(hh, fabs(a1), fabs(v[i])) + tiny;
            const int kq = (2 * i) & 3, kv = (2 * i + 1) & 3;
            if (fabs(eq) * mb[kq] > ma[kq] * dq) { ma[kq] = fabs(eq); mb[kq] = dq; }
            if (fabs(ev) * mb[kv] > ma[kv] * dv) { ma[kv] = fabs(ev); mb[kv] = dv; }
        }
#pragma unroll
        for (int k = 1; k < 4; ++k)
            if (ma[k] * mb[0] > ma[0] * mb[k]) { ma[0] = ma[k]; mb[0] = mb[k]; }
        const double err = ma[0] * rcp_fast(mb[0] * eps);
        const bool nanFlag = bad != 0;
        // adjustStep (rkck.cpp:100-113) with a call-free pow
        double hNew;
        bool accepted;
        if (err > 1.0 || !isfinite(err) || nanFlag) {
            accepted = false;
            hNew = (!isfinite(err) || nanFlag)
                       ? tol.p1 * hh
                       : fmax(tol.safety * hh * ctrl_pow_fast(err, tol.pshrnk), tol.p1 * hh);
        } else {
            accepted = true;
            const double hn =
                (err > tol.errcon) ? tol.safety * hh * ctrl_pow_fast(err, tol.pgrow) : 5.0 * hh;
            hNew = fmax(tol.h_min_floor, fmin(val(hMax), hn));
        }
        trace_step<(INSTR == 2)>(tol, true, t, h, 6, R(err), accepted);
        if (accepted) {
            t += h;
            stats_accept(st, hh);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                q[i] = Q[i];
                v[i] = Acc[i];
            }
            haveF = false;
            h = R(hNew);
            live = tEnd - t > R(tol.uround) * fabs_(tEnd);
        } else {
            ++st.steps_rejected;
            if (hNew < tol.h_min_floor) {  // freeze at the last accepted state
                st.underflow = 1;
                live = false;
            }
            h = R(hNew);
        }
        if (live && bud.spent_after(st)) live = false;
    }

    // error norm, controller and the accept/reject update of one attempt
    // Q/Acc: stage scratch, free here; FAST computes the candidate yNext into
    // them in the same pass as the error norm (one read of each stage slot)
    __device__ __forceinline__ void finish_attempt(const DevTol& tol, R (&Q)[M], R (&Acc)[M]) {
        using namespace ck;
        R* const q = y;
        R* const v = y + M;
        const R hMin(tol.h_min_floor);
        const R uround(tol.uround), eps(tol.eps), tiny(tol.tiny);
        // yErr folded into errorNorm (rkck.cpp:75-76, :88-98); the max is
        // order-independent, so the q and v halves are visited together
        R err;
        bool nanFlag = false;
        if constexpr (!is_exact<R>::value) {
            // FAST: h folded into the error weights; the max of |e_i| / d_i is
            // tracked as an argmax by cross-multiplication (no per-component
            // reciprocal) and divided out once; non-finite yErr components are
            // detected from their exponent fields
            const double hh = val(h);
            const double hd1 = hh * d1, hd3 = hh * d3, hd4 = hh * d4, hd5 = hh * d5, hd6 = hh * d6;
            double ma[4] = {0.0, 0.0, 0.0, 0.0}, mb[4] = {1.0, 1.0, 1.0, 1.0};
            const double hc1 = hh * c1, hc3 = hh * c3, hc4 = hh * c4, hc6 = hh * c6;
            int bad = 0;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double k0q = val(kget(0, i)), k1q = val(kget(1, i)), k2q = val(kget(2, i));
                const double k0v = val(Acc[i]), k1v = val(kget(1, M + i)),
                             k2v = val(kget(2, M + i));  // A6 = Acc (never stored)
                const double eq = fma(hd6, k0q, fma(hd5, val(kget(3, i)),
                                  fma(hd4, k2q, fma(hd3, k1q, hd1 * val(v[i])))));
                const double ev = fma(hd6, k0v, fma(hd5, val(kget(3, M + i)),
                                  fma(hd4, k2v, fma(hd3, k1v, hd1 * val(A0[i])))));
                // candidate yNext (rkck.cpp:74), kept only if the step is accepted
                Q[i] = R(fma(hc6, k0q, fma(hc4, k2q, fma(hc3, k1q, fma(hc1, val(v[i]), val(q[i]))))));
                Acc[i] = R(fma(hc6, k0v, fma(hc4, k2v, fma(hc3, k1v, fma(hc1, val(A0[i]), val(v[i]))))));
                bad |= ((__double2hiint(eq) & 0x7ff00000) == 0x7ff00000) |
                       ((__double2hiint(ev) & 0x7ff00000) == 0x7ff00000);
                const double dq = fma(hh, fabs(val(v[i])), fabs(val(q[i]))) + val(tiny);
                const double dv = fma(hh, fabs(val(A0[i])), fabs(val(v[i]))) + val(tiny);
                const int kq = (2 * i) & 3, kv = (2 * i + 1) & 3;
                if (fabs(eq) * mb[kq] > ma[kq] * dq) { ma[kq] = fabs(eq); mb[kq] = dq; }
                if (fabs(ev) * mb[kv] > ma[kv] * dv) { ma[kv] = fabs(ev); mb[kv] = dv; }
            }
#pragma unroll
            for (int k = 1; k < 4; ++k)
                if (ma[k] * mb[0] > ma[0] * mb[k]) { ma[0] = ma[k]; mb[0] = mb[k]; }
            nanFlag = bad != 0;
            err = R(ma[0] * rcp_fast(mb[0] * val(eps)));
        } else {
            // four interleaved accumulators: max and exact-argmax are associative,
            // so this only shortens the dependency chain (4x), never the result
            QuotMax qm[4];
            double fm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const R eq = h * (R(d1) * v[i] + R(d3) * kget(1, i) + R(d4) * kget(2, i) +
                                  R(d5) * kget(3, i) + R(d6) * kget(0, i));
                const R ev = h * (R(d1) * A0[i] + R(d3) * kget(1, M + i) +
                                  R(d4) * kget(2, M + i) + R(d5) * kget(3, M + i) +
                                  R(d6) * kget(0, M + i));
                if (!isfinite_(eq) || !isfinite_(ev)) nanFlag = true;
                const R dq = fabs_(q[i]) + fabs_(h * v[i]) + tiny;
                const R dv = fabs_(v[i]) + fabs_(h * A0[i]) + tiny;
                if constexpr (is_exact<R>::value) {
                    qm[(2 * i) & 3].push(fabs(val(eq)), val(dq));
                    qm[(2 * i + 1) & 3].push(fabs(val(ev)), val(dv));
                } else {
                    fm[(2 * i) & 3] = fmax(fm[(2 * i) & 3], fabs(val(eq)) * rcp_fast(val(dq)));
                    fm[(2 * i + 1) & 3] = fmax(fm[(2 * i + 1) & 3], fabs(val(ev)) * rcp_fast(val(dv)));
                }
            }
            qm[0].push(qm[1].a, qm[1].b);
            qm[2].push(qm[3].a, qm[3].b);
            qm[0].push(qm[2].a, qm[2].b);
            const double fmx = fmax(fmax(fm[0], fm[1]), fmax(fm[2], fm[3]));
            if constexpr (is_exact<R>::value)
                err = R(qm[0].value());
            else
                err = R(fmx);
            err = err / eps;
        }

        R hNew;
        bool accepted;
        if constexpr (is_exact<R>::value) {
            accepted = rkck_adjust(h, err, nanFlag, hMin, hMax, tol, hNew);
        } else {  // adjustStep (rkck.cpp:100-113) with a call-free pow
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
        trace_step<(INSTR == 2)>(tol, true, t, h, 6, err, accepted);
        if (accepted) {
            t += h;
            stats_accept(st, val(h));
            // yNext (rkck.cpp:74): the q half reads the old v, so it goes first
            if constexpr (is_exact<R>::value) {
#pragma unroll
                for (int i = 0; i < M; ++i)
                    q[i] = q[i] + h * (R(c1) * v[i] + R(c3) * kget(1, i) + R(c4) * kget(2, i) +
                                       R(c6) * kget(0, i));
#pragma unroll
                for (int i = 0; i < M; ++i)
                    v[i] = v[i] + h * (R(c1) * A0[i] + R(c3) * kget(1, M + i) +
                                       R(c4) * kget(2, M + i) + R(c6) * kget(0, M + i));
            } else {  // FAST: the candidate formed with the error norm
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    q[i] = Q[i];
                    v[i] = Acc[i];
                }
            }
            haveF = false;
            h = hNew;
            live = tEnd - t > uround * fabs_(tEnd);
        } else {
            ++st.steps_rejected;
            if (hNew < R(tol.h_min_floor)) {  // freeze at the last accepted state
                st.underflow = 1;
                live = false;
            }
            h = hNew;
        }
        if (live && bud.spent_after(st)) live = false;
    }
};

template <class P, class R, int INSTR>
__device__ __forceinline__ void rkck_nystrom_system(double t_in, double tEnd_in,
                                                    R (&y)[P::N], const R* g, const DevTol& tol,
                                                    DevStats& st) {
    NystromRkck<P, R, INSTR> s;
    s.gp = g;
#pragma unroll
    for (int c = 0; c < P::N; ++c) s.y[c] = y[c];
    s.start(t_in, tEnd_in, tol);
#pragma unroll 1
    while (s.live) s.attempt(tol);
#pragma unroll
    for (int c = 0; c < P::N; ++c) y[c] = s.y[c];
    st = s.st;
}

// Persistent-grid driver with dynamic refill (the north_star's ballot-bounded
// divergence): lanes claim systems from a global counter, one warp-aggregated
// atomicAdd per claim round; a lane whose system finishes stores it and
// claims the next, so a warp never idles behind its slowest system until the
// queue is empty. Results are per-system deterministic, hence independent of
// which lane integrates which system.
template <class P, class R, int INSTR>
__device__ __forceinline__ void rkck_nystrom_persistent(const double* __restrict__ y_in_unused,
                                                        double* __restrict__ y_soa,
                                                        DevStats* __restrict__ stats, long long num,
                                                        double t_in, double tEnd_in,
                                                        const DevTol& tol, int merge,
                                                        unsigned long long* counter,
                                                        int refill_min) {
    constexpr unsigned kFull = 0xffffffffu;
    const long long ld = tol.stride > 0 ? tol.stride : num;  // SoA row stride
    const unsigned lane = threadIdx.x & 31u;
    const unsigned lt_mask = (1u << lane) - 1u;
    NystromRkck<P, R, INSTR> s;
    long long sys = -1;
    bool has = false, exhausted = false;
    if (counter == nullptr) {  // static mapping: this lane's system, no refill
        exhausted = true;
        sys = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (sys < num) {
#pragma unroll
            for (int c = 0; c < P::N; ++c) s.y[c] = R(y_soa[sys + ld * (long long)c]);
            s.start(t_in, tEnd_in, tol);
            has = true;
        }
    }
    auto retire = [&]() {  // store a finished (or frozen) system and free the lane
#pragma unroll
        for (int c = 0; c < P::N; ++c) y_soa[sys + ld * (long long)c] = val(s.y[c]);
        if (stats != nullptr) {
            if (merge) {
                DevStats o = stats[sys];
                stats_merge(o, s.st);
                stats[sys] = o;
            } else {
                stats[sys] = s.st;
            }
        }
        has = false;
    };
#pragma unroll 1
    for (;;) {
        // refill round: idle lanes claim consecutive systems with one
        // warp-aggregated atomicAdd (loads of the claimed range stay coalesced)
        if (!exhausted) {
            const unsigned need = __ballot_sync(kFull, !has);
            if (need) {
                unsigned long long base = 0;
                const int leader = __ffs(need) - 1;
                if ((int)lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(need));
                base = __shfl_sync(kFull, base, leader);
                if (base + __popc(need) >= (unsigned long long)num) exhausted = true;
                if (!has) {
                    const unsigned long long mine = base + __popc(need & lt_mask);
                    if (mine < (unsigned long long)num) {
                        sys = (long long)mine;
#pragma unroll
                        for (int c = 0; c < P::N; ++c) s.y[c] = R(y_soa[sys + ld * (long long)c]);
                        s.start(t_in, tEnd_in, tol);
                        has = true;
                        if (!s.live) retire();  // empty interval: nothing to integrate
                    }
                }
            }
        }
        if (!__any_sync(kFull, has)) break;
        // attempts until refill_min lanes are idle (all of them once the queue
        // is exhausted): the same lean loop body as the static kernel, one
        // ballot per attempt
        const int stop = exhausted ? 32 : refill_min;
        // (running the attempt unguarded on idle lanes' stale state measured 2x
        // slower, so the attempt stays guarded by `has`)
#pragma unroll 1
        do {
            if (has && s.live) s.attempt(tol);
            if (has && !s.live) retire();
        } while (__popc(__ballot_sync(kFull, !has)) < stop);
    }
}

}  // namespace bode
