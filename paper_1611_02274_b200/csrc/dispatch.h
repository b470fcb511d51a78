// dispatch.h -- compiled-kernel registry shared by kernels.cu and host.cu.
#pragma once

#include <cuda_runtime.h>

namespace bode {

constexpr int kMaxBlock = 256;

// One attempt of the traced system (bode_step_record_t, the reference's
// StepRecord, ode_problem.hpp:85-91).
struct StepRec {
    double t, h, err;
    int stages, accepted;
};
static_assert(sizeof(StepRec) == 32, "StepRec must match bode_step_record_t");

struct DevTol {  // bode_tol_t, by value in the kernel parameters
    double eps, abs_tol, rel_tol, uround, tiny, safety, p1, errcon, pgrow, pshrnk,
        h_min_floor, kappa;
    const double* powtab;    // host-libm pow tables on this device (arith.cuh), or null
    const double* rkc_coef;  // RKC coefficient table for this kappa/policy (rkc.cuh), or null
    int refill_min;          // persistent kernels: idle lanes that trigger a refill round
    long long stride;        // SoA row stride of y and g in doubles (0: the launch's num),
                             // so a launch can cover a column range of a larger batch
    int dim;                 // the problem's dimension (run-time-dimension kernels, wide.cuh)
    double* scratch;         // wide.cuh: per-block vector scratch in global memory, or null
    long long max_attempts;  // per-window attempt budget per system (0: none)
    StepRec* trace;                  // per-attempt records of a one-system launch, or null
    long long trace_cap;
    unsigned long long* trace_count;
};

struct DevStats {  // bode_stats_t, per system (AoS, 64 bytes)
    long long steps_accepted, steps_rejected, rhs_evals, spec_rad_evals, stages_total;
    double h_min_seen, h_max_seen;
    int underflow, budget_exhausted;
};
static_assert(sizeof(DevStats) == 64, "DevStats must match bode_stats_t");

template <class P, int L>
constexpr int C_of() { return P::N / L; }

// One-system-per-block kernels (wide.cuh): state-length vectors per system,
// threads per block (upper bound), and the largest vector set kept in
// shared memory (beyond it the vectors live in a per-block global scratch).
constexpr int kWideVecs = 8;
constexpr int kWideMaxBlock = 512;
constexpr int kWideSmemMax = 200 * 1024;
// threads per block for dimension n: one component per thread up to
// kWideMaxBlock, in whole warps
__host__ __device__ constexpr int wide_block(int n) {
    return n >= kWideMaxBlock ? kWideMaxBlock : ((n + 31) / 32) * 32;
}

// Launchers return the launching runtime's cudaGetLastError() as an int.
using LaunchFn = int (*)(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          const double* g, double* y, DevStats* st, long long num, double t,
                          double tEnd, DevTol tol, int merge);

using LaunchPersistentFn = int (*)(const void* fn, dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t s, const double* g, double* y, DevStats* st,
                                    long long num, double t, double tEnd, DevTol tol, int merge,
                                    unsigned long long* counter);

struct KernelEntry {
    int kind, dim, param_dim, solver, arith;
    int lanes;            // lanes per system (L)
    int maxreg;           // register cap of this instance (0: ptxas default, up to 255)
    int smem_per_thread;  // dynamic shared memory bytes per thread
    int default_block;
    const void* fn;
    LaunchFn launch;
    int (*build_rkc_table)(double* tab, double kappa, cudaStream_t s);  // null for RKCK
    // persistent variant with dynamic refill (null if none): a grid sized to the
    // resident capacity whose lanes claim systems from `counter`
    const void* pfn = nullptr;
    LaunchPersistentFn launch_persistent = nullptr;
    // Makes `device` current and raises fn's dynamic shared-memory limit to
    // smem_bytes, in the CUDA runtime of the translation unit that compiled the
    // kernel (a problem registered from another library carries its own).
    int (*prepare)(const void* fn, int device, int smem_bytes) = nullptr;
    // fixed-step harness (integrateFixed) for this problem/solver/policy
    const void* ffn = nullptr;
    int (*launch_fixed)(const void* fn, dim3 grid, dim3 block, cudaStream_t s, const double* g,
                         double* y, long long num, double t0, double tEnd, long long numSteps,
                         long long stages, double kappa) = nullptr;
    // 1: one system per thread block for any dimension (wide.cuh), dim == 0;
    // chosen when no lane-group kernel is compiled for the problem's dim
    int wide = 0;
    // instances with the attempt-budget check (bode_set_attempt_budget), launched
    // in place of fn / pfn while a budget is set
    const void* bfn = nullptr;
    const void* bpfn = nullptr;
    // run-time-dimension lane kernels (problems.cuh is_runtime_dim, dim == 0):
    // the largest dimension they hold; chosen when no exact-dim kernel exists
    int cap = 0;
    // one-system-per-block fixed-step harness (wide entries; ffn is its kernel)
    int (*launch_fixed_wide)(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             const double* g, double* y, long long num, double t0, double tEnd,
                             long long numSteps, long long stages, double kappa, int dim,
                             double* scratch) = nullptr;
};

const KernelEntry* kernel_table(int* count);

// repack.cu: cost-aware re-packing of a device-resident batch
int repack_by_cost(int N, int P, long long num, double* y, double* g, DevStats* st,
                   long long* order, cudaStream_t s);
int repack_by(int N, int P, long long num, double* y, double* g, DevStats* st, long long* order,
              int param_row, cudaStream_t s);
int unpack(int N, int P, long long num, double* y, double* g, DevStats* st, long long* order,
           double* y_out, cudaStream_t s);
int init_order(long long* order, long long num, cudaStream_t s);
int lockstep_efficiency(const DevStats* st, long long num, int group, double* eff,
                        cudaStream_t s);
const double* device_powtab();
long long rkc_table_doubles();

}  // namespace bode
