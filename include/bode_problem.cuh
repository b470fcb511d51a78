// bode_problem.cuh -- user problems for the device integrators.
//
// The reference integrates any OdeProblem {dim, paramDim, rhs}
// (proj/include/batchode/ode_problem.hpp:22-30); the paper's GPU code takes a
// user-supplied __device__ dydt compiled into the integration kernel
// (PAPER.md:370, :416). Here a problem is a struct compiled into the RKCK and
// RKC kernels, so its right-hand side is fused with the stage arithmetic and
// stays in registers:
//
//   struct MyProblem {
//       static constexpr int N = ...;   // state dimension
//       static constexpr int P = ...;   // per-system parameters (0 if none)
//       // this lane's slice dy[c] = f(t, y)[G.lane * (N / L) + c] of the RHS;
//       // y[c] likewise; g[0..P) are the system's parameters. Lanes of the
//       // group exchange halo values with G.from / G.from_prev / G.from_next.
//       // Every lane must reach each of these calls (no data-dependent
//       // branch around them): RKC on lane groups calls rhs warp-uniformly
//       // with a full-warp shuffle mask (rkc.cuh).
//       template <class R, int L>
//       __device__ static void rhs(const bode::Group<L>& G, R t, const R (&y)[N / L],
//                                  const R* g, R (&dy)[N / L]);
//   };
//   BODE_REGISTER_PROBLEM(my_problem, MyProblem, BODE_PROBLEM_USER_BASE + 0, 1, 1)
//
// Second-order systems (q' = v, v' = a(t, q; g)) derive from
// bode::SecondOrderProblem<Self, dim(q), P> and provide only
//   template <class R> __device__ static void accel(R t, const R* q, const R* g, R* a);
// RKCK then runs the Nystrom kernels (one lane per system; FAST in
// Runge-Kutta-Nystrom form, the fastest path in this library).
//
// R is bode::xd under the EXACT policy -- every + - * / is one IEEE binary64
// operation, so written in the host code's expression order the device result
// is bitwise the host's -- and double under FAST (FMA contraction allowed).
// Use bode::sqrt_, fabs_, fmax_, ... for R-generic math.
//
// Compile with nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17
// -I<repo>/include into a shared library linked against libbode.so; loading
// it registers the kernels (bode_register_kernels), after which
// bode_int_driver / bode_outer_loop / bode_int_driver_device accept the kind.
#pragma once

#include "bode.h"
#include "../paper_1611_02274_b200/csrc/kernel_entry.cuh"

namespace bode {

// RKCK keeps its four stage slots in shared memory once a lane's slice is
// large enough that registers would spill (rkck.cuh KStore).
template <class P, int L>
constexpr bool kUserKsmem = (P::N / L) > 8;

// The kernel entries of one problem: RKCK with RKCK_L lanes per system and
// RKC with RKC_L lanes, each under both arithmetic policies.
template <class P, int RKCK_L, int RKC_L, int MAXREG = 0>
struct UserEntries {
    static_assert(P::N % RKCK_L == 0 && P::N % RKC_L == 0, "lanes must divide N");
    static_assert(32 % RKCK_L == 0 && 32 % RKC_L == 0, "lanes must divide the warp");
    KernelEntry e[4];
    explicit UserEntries(int kind)
        : e{make_entry<P, xd, RKCK_L, 0, kUserKsmem<P, RKCK_L>, MAXREG>(kind, BODE_ARITH_EXACT),
            make_entry<P, double, RKCK_L, 0, kUserKsmem<P, RKCK_L>, MAXREG>(kind, BODE_ARITH_FAST),
            make_entry<P, xd, RKC_L, 1, false, MAXREG>(kind, BODE_ARITH_EXACT),
            make_entry<P, double, RKC_L, 1, false, MAXREG>(kind, BODE_ARITH_FAST)} {}
};

}  // namespace bode

// Compiles the problem's kernels in this translation unit and registers them
// with libbode when the enclosing library is loaded. NAME is an identifier;
// the _R form caps registers per thread (e.g. 128 for 16 warps/SM).
#define BODE_REGISTER_PROBLEM_R(NAME, TYPE, KIND, RKCK_LANES, RKC_LANES, MAXREG)             \
    namespace {                                                                             \
    const int bode_registered_##NAME = [] {                                                \
        static const bode::UserEntries<TYPE, RKCK_LANES, RKC_LANES, MAXREG> entries(KIND);  \
        return bode_register_kernels(entries.e, 4, (int32_t)sizeof(bode::KernelEntry));     \
    }();                                                                                    \
    }
#define BODE_REGISTER_PROBLEM(NAME, TYPE, KIND, RKCK_LANES, RKC_LANES) \
    BODE_REGISTER_PROBLEM_R(NAME, TYPE, KIND, RKCK_LANES, RKC_LANES, 0)
