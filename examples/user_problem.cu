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
#include <cmath>

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

// A second-order problem: the gravitational N-body problem in 3-D with
// per-system masses (params 0..NB-1), y = (positions, velocities). Declaring
// it through bode::SecondOrderProblem gives RKCK the Nystrom kernels (FAST in
// Runge-Kutta-Nystrom form). The host form is bode_example_nbody_rhs.
struct NBody3 : bode::SecondOrderProblem<NBody3, 3 * 5, 5> {
    static constexpr int NB = 5;
    template <class R>
    __device__ __forceinline__ static void accel(R, const R* q, const R* m, R* a) {
#pragma unroll
        for (int k = 0; k < 3 * NB; ++k) a[k] = R(0.0);
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int j = i + 1; j < NB; ++j) {
                const R dx = q[3 * j] - q[3 * i];
                const R dy = q[3 * j + 1] - q[3 * i + 1];
                const R dz = q[3 * j + 2] - q[3 * i + 2];
                const R r2 = dx * dx + dy * dy + dz * dz;
                const R inv = R(1.0) / (r2 * bode::sqrt_(r2));
                a[3 * i] += m[j] * dx * inv;
                a[3 * i + 1] += m[j] * dy * inv;
                a[3 * i + 2] += m[j] * dz * inv;
                a[3 * j] -= m[i] * dx * inv;
                a[3 * j + 1] -= m[i] * dy * inv;
                a[3 * j + 2] -= m[i] * dz * inv;
            }
    }
};

BODE_REGISTER_PROBLEM(nbody3, NBody3, BODE_PROBLEM_USER_BASE + 97, 1, 1)

extern "C" void bode_example_nbody_rhs(double, const double* y, const double* m, double* dy) {
    const int nb = 5, M = 3 * nb;
    for (int k = 0; k < M; ++k) dy[k] = y[M + k];
    double* a = dy + M;
    for (int k = 0; k < M; ++k) a[k] = 0.0;
    for (int i = 0; i < nb; ++i)
        for (int j = i + 1; j < nb; ++j) {
            const double dx = y[3 * j] - y[3 * i];
            const double dy_ = y[3 * j + 1] - y[3 * i + 1];
            const double dz = y[3 * j + 2] - y[3 * i + 2];
            const double r2 = dx * dx + dy_ * dy_ + dz * dz;
            const double inv = 1.0 / (r2 * std::sqrt(r2));
            a[3 * i] += m[j] * dx * inv;
            a[3 * i + 1] += m[j] * dy_ * inv;
            a[3 * i + 2] += m[j] * dz * inv;
            a[3 * j] -= m[i] * dx * inv;
            a[3 * j + 1] -= m[i] * dy_ * inv;
            a[3 * j + 2] -= m[i] * dz * inv;
        }
}
