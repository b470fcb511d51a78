// user_problem.cu -- an out-of-tree problem library: the user-supplied dydt
// of the paper compiled into the device RKCK/RKC kernels
// through include/bode_problem.cuh, registered with libbode when this library
// is loaded.
//
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -shared
//              -Xcompiler -fPIC -Iinclude examples/user_problem.cu
//              -Lpaper_1611_02274_b200/lib -lbode -o libuser_problem.so
//   use:   load libbode, then this library (ctypes.CDLL / dlopen); kind
//          BODE_PROBLEM_USER_BASE + 96 is then accepted by every entry point.
//
// The problem: Lorenz-96, y_i' = (y_{i+1} - y_{i-2}) y_{i-1} - y_i + F with
// cyclic indices, N = 40, forcing F per system (param 0). The host form below
// (bode_example_lorenz96_rhs) is what the reference's drivers integrate in the
// parity tests; the device form is the same expression in the same order.
#include "bode_problem.cuh"

struct Lorenz96 {
    static constexpr int N = 40, P = 1;
    template <class R, int L>
    __device__ __forceinline__ static void rhs(const bode::Group<L>&, R, const R (&y)[N / L],
                                               const R* g, R (&dy)[N / L]) {
        static_assert(L == 1, "cyclic coupling: one lane per system");
        const R F = g[0];
#pragma unroll
        for (int i = 0; i < N; ++i)
            dy[i] = (y[(i + 1) % N] - y[(i + N - 2) % N]) * y[(i + N - 1) % N] - y[i] + F;
    }
};

BODE_REGISTER_PROBLEM(lorenz96, Lorenz96, BODE_PROBLEM_USER_BASE + 96, 1, 1)

// Host form for the reference's OdeProblem::rhs (test oracle).
extern "C" void bode_example_lorenz96_rhs(double, const double* y, const double* g, double* dy) {
    const int n = 40;
    const double F = g[0];
    for (int i = 0; i < n; ++i)
        dy[i] = (y[(i + 1) % n] - y[(i + n - 2) % n]) * y[(i + n - 1) % n] - y[i] + F;
}
