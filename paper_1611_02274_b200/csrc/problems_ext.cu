// problems_ext.cu -- problems beyond the reference's set, built through the
// public user-problem interface (include/bode_problem.cuh) exactly as an
// out-of-tree library would be, and registered when libbode loads.
//
// Brusselator: 1-D reaction-diffusion of the autocatalytic Brusselator
// mechanism (a chemical-kinetics RHS with diffusion, the moderately stiff
// workload RKC is designed for; the paper's motivating use is chemical
// kinetics):
//   u' = A + u^2 v - (B + 1) u + alpha (u_{i-1} - 2u_i + u_{i+1}) / dx^2
//   v' = B u - u^2 v        + alpha (v_{i-1} - 2v_i + v_{i+1}) / dx^2
// on n interior points, dx = 1/(n+1), boundary values (A, B/A), per-system
// parameters g = (A, B, alpha) -- so stiffness varies per system with alpha.
// State interleaved y = (u_1, v_1, ..., u_n, v_n): a lane's slice holds whole
// grid points, and the halo is one (u, v) pair from each neighbouring lane.
// The host form that the reference drivers integrate for the parity tests is
// in oracle/ref_shim.cpp (same expression order).
#include "../../include/bode_problem.cuh"

namespace bode {

template <int NN>
struct Brusselator {
    static constexpr int N = 2 * NN, P = 3;
    static constexpr const char* name = "brusselator";
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const Group<L>& G, R, const R (&y)[N / L],
                                               const R* g, R (&out)[N / L]) {
        constexpr int C = N / L;
        static_assert(C % 2 == 0, "a lane holds whole (u, v) grid points");
        const R A = g[0], B = g[1], alpha = g[2];
        const R dx = R(1.0) / R(double(NN + 1));
        const R c = alpha / (dx * dx);
        const R ub = A, vb = B / A;
        const R Bp1 = B + R(1.0);
        const R uLh = R(G.from_prev(val(y[C - 2]))), vLh = R(G.from_prev(val(y[C - 1])));
        const R uRh = R(G.from_next(val(y[0]))), vRh = R(G.from_next(val(y[1])));
        const bool first = G.lane == 0, last = G.lane == L - 1;
#pragma unroll
        for (int k = 0; k < C / 2; ++k) {
            const R u = y[2 * k], v = y[2 * k + 1];
            const R uL = k > 0 ? y[2 * k - 2] : (first ? ub : uLh);
            const R vL = k > 0 ? y[2 * k - 1] : (first ? vb : vLh);
            const R uR = k < C / 2 - 1 ? y[2 * k + 2] : (last ? ub : uRh);
            const R vR = k < C / 2 - 1 ? y[2 * k + 3] : (last ? vb : vRh);
            const R uuv = u * u * v;
            out[2 * k] = A + uuv - Bp1 * u + c * (uL - R(2.0) * u + uR);
            out[2 * k + 1] = B * u - uuv + c * (vL - R(2.0) * v + vR);
        }
    }
};

}  // namespace bode

// n = 32 grid points (dim 64): RKC with 4 lanes per system, uncapped (8 warps/SM);
// RKCK candidates (lanes x register cap) registered in
// preference order, selectable with BODE_LANES / BODE_MAXREG for A/B runs
namespace {
using Bru = bode::Brusselator<32>;
const int bode_registered_brusselator32 = [] {
    static const bode::KernelEntry e[] = {
        // RKC EXACT measured (2^20 systems, 5 windows, system-windows/s): 4 lanes
        // uncapped 6.33e7, 8 @128 6.07e7, 4 @168 5.83e7, 8 @168 5.58e7 (r01cq);
        // 4 @224 in 32-thread blocks 5.78e7, 4 @200 in 64-thread blocks 5.89e7 (r01df);
        // the heavier reaction RHS and 3 instead of 7 sum hand-offs favour 4 lanes
        bode::make_entry<Bru, bode::xd, 4, 1, false, 0>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_EXACT),
        bode::make_entry<Bru, double, 4, 1, false, 0>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_FAST),
        bode::make_entry<Bru, bode::xd, 8, 1, false, 128>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_EXACT),
        bode::make_entry<Bru, double, 8, 1, false, 128>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_FAST),
        // RKCK FAST measured (2^20 systems, 5 windows, FP64 fraction): 8 lanes @128
        // 0.490, 4 @255 0.483, 8 @255 0.437, 16 @128 0.410, 4 @128 0.326
        bode::make_entry<Bru, double, 8, 0, true, 128>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_FAST),
        bode::make_entry<Bru, bode::xd, 8, 0, true, 128>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_EXACT),
        bode::make_entry<Bru, bode::xd, 4, 0, true, 0>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_EXACT),
        bode::make_entry<Bru, double, 4, 0, true, 0>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_FAST),
        bode::make_entry<Bru, double, 16, 0, true, 128>(BODE_PROBLEM_BRUSSELATOR, BODE_ARITH_FAST),
    };
    return bode_register_kernels(e, (int32_t)(sizeof(e) / sizeof(e[0])),
                                 (int32_t)sizeof(bode::KernelEntry));
}();
}  // namespace
