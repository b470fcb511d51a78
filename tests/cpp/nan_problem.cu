// nan_problem.cu -- the device form of the right-hand side that
// test_batch.cpp:241-258 builds from a host lambda: y' = NaN for a system
// whose parameter g0 exceeds 0.5, else y' = -y. Registered with libbode when
// this test library is loaded (include/bode_problem.cuh), so the transcribed
// reference test (test_batch_dropin.cpp) can take it as an OdeProblem.
#include "bode_problem.cuh"

struct NanGate {
    static constexpr int N = 1, P = 1;
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const bode::Group<L>&, R, const R (&y)[1],
                                               const R* g, R (&dy)[1]) {
        dy[0] = bode::val(g[0]) > 0.5 ? R(__longlong_as_double(0x7ff8000000000000LL)) : -y[0];
    }
};

BODE_REGISTER_PROBLEM(nan_gate, NanGate, BODE_PROBLEM_USER_BASE + 500, 1, 1)
