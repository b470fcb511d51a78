// kernel_entry.cuh -- the intDriver kernel templates and
// their dispatch-table entries, shared by the built-in table (kernels.cu) and
// by problems registered through include/bode_problem.cuh.
//
// One lane group (L lanes) integrates one system over one window [t, tEnd]:
// coalesced SoA load of y[i + num*j] (batch.hpp:15-29), the
// fused solver (rkck*.cuh / rkc.cuh), SoA store, per-system stats (AoS).
// All arithmetic is FP64 on the CUDA cores; nothing here is a contraction,
// so there are no tensor cores on this path.
#pragma once

#include <cuda_runtime.h>

#include "dispatch.h"
#include "rkc.cuh"
#include "rkck_nystrom.cuh"
#include "rkck_pleiades2.cuh"
#include "fixed.cuh"
#include "wide.cuh"

namespace bode {

// Parameter slots a kernel holds per system: the problem's own, or the
// kernel-generated n and constant of a run-time-dimension problem.
template <class P>
__host__ __device__ constexpr int params_of() {
    if constexpr (is_runtime_dim<P>::value)
        return P::PG;
    else
        return P::P > 0 ? P::P : 1;
}

// Global component held by lane `lane` of a group in local slot c. Blocks of
// C consecutive components by default; the 2-lane Pleiades split is by axis:
// lane l holds positions [7l, 7l+7) and velocities [14+7l, 14+7l+7).
template <class P, int L>
__device__ __forceinline__ int comp_index(int lane, int c) {
    constexpr int C = P::N / L;
    if constexpr (is_pleiades<P> && L == 2)
        return c < 7 ? 7 * lane + c : 14 + 7 * lane + (c - 7);
    else
        return lane * C + c;
}

// blockIdx.x * blockDim.x + threadIdx.x, read afresh (see integrate_kernel)
__device__ __forceinline__ long long fresh_thread_index() {
    unsigned tid, ctaid, ntid;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
    asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(ctaid));
    asm volatile("mov.u32 %0, %%ntid.x;" : "=r"(ntid));
    return (long long)ctaid * ntid + tid;
}

// MAXREG > 0 caps registers per thread (__maxnreg__) to reach a target
// occupancy; 0 leaves ptxas the full 255 (launch bound kMaxBlock threads).
template <class P, class R, int L, int SOLVER, bool KSMEM, int MAXREG, int INSTR>
__global__ void __maxnreg__(MAXREG > 0 ? MAXREG : 255)
    integrate_kernel(const double* __restrict__ g_soa, double* __restrict__ y_soa,
                     DevStats* __restrict__ stats, long long num, double t, double tEnd,
                     DevTol tol, int merge) {
    constexpr int C = P::N / L;
    constexpr int PP = params_of<P>();
    const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long sys = gt / L;
    // RKC on lane groups runs warp-uniform (rkc.cuh): lanes past the batch's
    // end stay with their warp as idle groups; elsewhere lanes retire here
    constexpr bool kUniform = SOLVER == 1 && L > 1;
    const bool inRange = sys < num;
    if (kUniform ? !__any_sync(0xffffffffu, inRange) : !inRange) return;
    const long long ld = tol.stride > 0 ? tol.stride : num;  // SoA row stride
    Group<L> G(kUniform);
    R y[C];
    R g[PP];
    const int n = is_runtime_dim<P>::value ? tol.dim : P::N;  // components held (the rest pad)
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int ci = comp_index<P, L>(G.lane, c);
        y[c] = R(inRange && ci < n ? y_soa[sys + ld * (long long)ci] : 0.0);
    }
#pragma unroll
    for (int p = 0; p < PP; ++p)
        g[p] = R(P::P > 0 && inRange ? g_soa[sys + ld * (long long)p] : 0.0);
    if constexpr (is_runtime_dim<P>::value) {
        double gg[2];
        P::params(n, gg);
        g[0] = R(gg[0]);
        g[1] = R(gg[1]);
    }
    DevStats st;
    if constexpr (SOLVER == 0 && is_pleiades<P> && L == 2)
        rkck_pleiades2_system<R, INSTR>(G, t, tEnd, y, tol, st);
    else if constexpr (SOLVER == 0 && is_second_order<P>::value && L == 1)
        rkck_nystrom_system<P, R, INSTR>(t, tEnd, y, g, tol, st);
    else if constexpr (SOLVER == 0)
        rkck_system<P, R, L, KSMEM, INSTR>(G, t, tEnd, y, g, tol, st);
    else if constexpr (L == 1)
        rkc_system_lane<P, R, INSTR>(G, t, tEnd, y, g, tol, st);
    else
        rkc_system<P, R, L, INSTR>(G, inRange, t, tEnd, y, g, tol, st);
    // RKC lane groups: the system index again from the special registers
    // (volatile reads, so it is recomputed here rather than kept live -- and
    // spilled -- across the whole integration; the heat kernels' last spills).
    const long long sys_out = kUniform ? fresh_thread_index() / L : sys;
    if (kUniform ? sys_out >= num : !inRange) return;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int ci = comp_index<P, L>(G.lane, c);
        if (ci < n) y_soa[sys_out + ld * (long long)ci] = val(y[c]);
    }
    if (stats != nullptr && G.lane == 0) {
        if (merge) {
            DevStats o = stats[sys_out];
            stats_merge(o, st);
            stats[sys_out] = o;
        } else {
            stats[sys_out] = st;
        }
    }
}

// Persistent-grid RKCK for second-order problems, one lane per system.
template <class P, class R, int INSTR>
__global__ void __launch_bounds__(kMaxBlock)
    persistent_kernel(const double* __restrict__ g_soa, double* __restrict__ y_soa,
                      DevStats* __restrict__ stats, long long num, double t, double tEnd,
                      DevTol tol, int merge, unsigned long long* counter) {
    rkck_nystrom_persistent<P, R, INSTR>(g_soa, y_soa, stats, num, t, tEnd, tol, merge, counter,
                                  tol.refill_min);
}

// ---- dispatch table ----
template <class P, class R, int L, int SOLVER, bool KSMEM, int MAXREG>
static KernelEntry make_entry(int kind, int arith) {
    KernelEntry e;
    e.kind = kind;
    e.dim = is_runtime_dim<P>::value ? 0 : P::N;
    e.cap = is_runtime_dim<P>::value ? P::N : 0;
    e.param_dim = P::P;
    e.solver = SOLVER;
    e.arith = arith;
    e.lanes = L;
    e.maxreg = MAXREG;
    if constexpr (SOLVER == 0 && is_second_order<P>::value && L == 1)
        e.smem_per_thread = nystrom_smem_doubles<P, R>() * (int)sizeof(double);
    else
        e.smem_per_thread = SOLVER == 1 ? kRkcSmemStride<C_of<P, L>(), L>() * (int)sizeof(double)
                            : KSMEM     ? kSmemStride<C_of<P, L>()>() * (int)sizeof(double)
                                        : 0;
    // Instances: 0 plain (the default launch), 2 instrumented (attempt budget
    // and step trace), launched only while a budget or a trace is requested.
#ifndef BODE_RKN_BUDGET_INSTANCE
#define BODE_RKN_BUDGET_INSTANCE 1
#endif
    // The FAST one-lane Pleiades (RKN) kernel defaults to instance 1 (budget
    // countdown, no trace): ptxas allocates it without spills at 254 registers,
    // the plain one with 76 bytes of spills at 255 (+0.4%, r02y); without a
    // budget the countdown never fires.
    if constexpr (BODE_RKN_BUDGET_INSTANCE && SOLVER == 0 && is_pleiades<P> && L == 1 &&
                  !is_exact<R>::value)
        e.fn = (const void*)&integrate_kernel<P, R, L, SOLVER, KSMEM, MAXREG, 1>;
    else
        e.fn = (const void*)&integrate_kernel<P, R, L, SOLVER, KSMEM, MAXREG, 0>;
    e.bfn = (const void*)&integrate_kernel<P, R, L, SOLVER, KSMEM, MAXREG, 2>;
    e.launch = [](const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                  const double* g, double* y, DevStats* st, long long num, double t,
                  double tEnd, DevTol tol, int merge) -> int {
        auto k = (void (*)(const double*, double*, DevStats*, long long, double, double, DevTol,
                           int))fn;
        k<<<grid, block, smem, s>>>(g, y, st, num, t, tEnd, tol, merge);
        return (int)cudaGetLastError();
    };
    e.default_block = KSMEM ? 128 : 128;
    e.prepare = [](const void* fn, int device, int smem_bytes) -> int {
        cudaError_t err = cudaSetDevice(device);
        if (err == cudaSuccess && smem_bytes > 48 * 1024)
            err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
        return (int)err;
    };
    e.build_rkc_table = nullptr;
    // (run-time-dimension problems take the one-system-per-block fixed-step kernels)
    if constexpr (!(SOLVER == 0 && is_pleiades<P> && L == 2) && !is_runtime_dim<P>::value) {
        e.ffn = (const void*)&fixed_kernel<P, R, L, SOLVER>;
        e.launch_fixed = [](const void* fn, dim3 grid, dim3 block, cudaStream_t s,
                            const double* g, double* y, long long num, double t0, double tEnd,
                            long long numSteps, long long stages, double kappa) -> int {
            auto k = (void (*)(const double*, double*, long long, double, double, long long,
                               long long, double))fn;
            k<<<grid, block, 0, s>>>(g, y, num, t0, tEnd, numSteps, stages, kappa);
            return (int)cudaGetLastError();
        };
    }
    if constexpr (SOLVER == 0 && is_second_order<P>::value && L == 1 && P::P == 0) {
        // (routing static launches through this instance with counter == nullptr
        // removes the spills but measured 9% slower: the any_sync loop costs more)
        e.pfn = (const void*)&persistent_kernel<P, R, 0>;
        e.bpfn = (const void*)&persistent_kernel<P, R, 2>;
        e.launch_persistent = [](const void* fn, dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t s, const double* g, double* y, DevStats* st,
                                 long long num, double t, double tEnd, DevTol tol, int merge,
                                 unsigned long long* counter) -> int {
            auto k = (void (*)(const double*, double*, DevStats*, long long, double, double,
                               DevTol, int, unsigned long long*))fn;
            k<<<grid, block, smem, s>>>(g, y, st, num, t, tEnd, tol, merge, counter);
            return (int)cudaGetLastError();
        };
    }
    if constexpr (SOLVER == 1)
        e.build_rkc_table = [](double* tab, double kappa, cudaStream_t s) -> int {
            rkc_coef_table_kernel<R><<<(unsigned)((kRkcTableMaxS + 63) / 64), 64, 0, s>>>(tab, kappa);
            return (int)cudaGetLastError();
        };
    return e;
}

// One system per thread block for a problem with a run-time dimension
// (wide.cuh); matched by kind when no lane-group kernel fits the dim.
template <class Prob, class R, int SOLVER>
static KernelEntry make_wide_entry(int kind, int arith) {
    KernelEntry e;
    e.kind = kind;
    e.dim = 0;
    e.param_dim = Prob::P;
    e.solver = SOLVER;
    e.arith = arith;
    e.lanes = 32;  // one group per warp for the lockstep-efficiency check
    e.maxreg = 0;
    e.smem_per_thread = 0;
    e.default_block = 0;
    e.wide = 1;
    e.fn = (const void*)&wide_kernel<Prob, R, SOLVER>;
    e.bfn = e.fn;  // the block kernels always carry the (cheap, per-block) check
    e.ffn = (const void*)&wide_fixed_kernel<Prob, R, SOLVER>;
    e.launch_fixed_wide = [](const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             const double* g, double* y, long long num, double t0, double tEnd,
                             long long numSteps, long long stages, double kappa, int dim,
                             double* scratch) -> int {
        auto k = (void (*)(const double*, double*, long long, double, double, long long,
                           long long, double, int, double*))fn;
        k<<<grid, block, smem, s>>>(g, y, num, t0, tEnd, numSteps, stages, kappa, dim, scratch);
        return (int)cudaGetLastError();
    };
    e.launch = [](const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                  const double* g, double* y, DevStats* st, long long num, double t,
                  double tEnd, DevTol tol, int merge) -> int {
        auto k = (void (*)(const double*, double*, DevStats*, long long, double, double, DevTol,
                           int))fn;
        k<<<grid, block, smem, s>>>(g, y, st, num, t, tEnd, tol, merge);
        return (int)cudaGetLastError();
    };
    e.prepare = [](const void* fn, int device, int smem_bytes) -> int {
        cudaError_t err = cudaSetDevice(device);
        if (err == cudaSuccess && smem_bytes > 48 * 1024)
            err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
        return (int)err;
    };
    e.build_rkc_table = nullptr;
    if constexpr (SOLVER == 1)
        e.build_rkc_table = [](double* tab, double kappa, cudaStream_t s) -> int {
            rkc_coef_table_kernel<R><<<(unsigned)((kRkcTableMaxS + 63) / 64), 64, 0, s>>>(tab, kappa);
            return (int)cudaGetLastError();
        };
    return e;
}

#define BODE_BOTH_ARITH_R(P, L, SOLVER, KSMEM, KIND, MAXREG)                  \
    make_entry<P, xd, L, SOLVER, KSMEM, MAXREG>(KIND, 0),                    \
        make_entry<P, double, L, SOLVER, KSMEM, MAXREG>(KIND, 1)
#define BODE_BOTH_ARITH(P, L, SOLVER, KSMEM, KIND) BODE_BOTH_ARITH_R(P, L, SOLVER, KSMEM, KIND, 0)

}  // namespace bode
