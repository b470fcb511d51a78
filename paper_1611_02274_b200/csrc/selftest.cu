// selftest.cu -- diagnostics exported through the C ABI (bode_selftest_*).
#include <cuda_runtime.h>

#include <string>

#include "../../include/bode.h"
#include "arith.cuh"
#include "dispatch.h"

namespace {

__global__ void cbrt_kernel(const double* __restrict__ x, double* __restrict__ out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = bode::glibc_cbrt(x[i]);
}

}  // namespace

extern "C" int bode_selftest_cbrt(const double* x, double* out, int64_t n) {
    if (n < 1 || x == nullptr || out == nullptr) return BODE_E_INVALID_SHAPE;
    int dev = 0;
    if (cudaGetDeviceCount(&dev) != cudaSuccess || dev < 1) {
        cudaGetLastError();
        return BODE_E_NO_DEVICE;
    }
    double *dx = nullptr, *dy = nullptr;
    if (cudaMalloc(&dx, n * sizeof(double)) != cudaSuccess) return BODE_E_CUDA;
    if (cudaMalloc(&dy, n * sizeof(double)) != cudaSuccess) {
        cudaFree(dx);
        return BODE_E_CUDA;
    }
    cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice);
    cbrt_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dx, dy, n);
    cudaError_t e = cudaMemcpy(out, dy, n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    return e == cudaSuccess ? BODE_OK : BODE_E_CUDA;
}

namespace {

// 8 independent DFMA chains per thread keep the FP64 pipe saturated
// regardless of its latency; values stay bounded (x <- x*a + b, |a| < 1).
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains live
}

}  // namespace

// Measured FP64 FMA throughput of the current device: flop/s (2 per DFMA).
extern "C" int bode_selftest_fp64_peak(double* flops_per_s, double* seconds) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return BODE_E_NO_DEVICE;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, 65536 * sizeof(double)) != cudaSuccess) return BODE_E_CUDA;
    const int blocks = sms * 8, threads = 256, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_peak_kernel<<<blocks, threads>>>(out, 64, 0.999, 1e-3);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_peak_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return BODE_E_CUDA;
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    *seconds = best * 1e-3;
    *flops_per_s = flops / (*seconds);
    return BODE_OK;
}

namespace {
__global__ void pow_kernel(const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ out, long long n, const double* T) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = bode::pow_glibc(x[i], y[i], T);
}
}  // namespace

extern "C" int bode_selftest_pow(const double* x, const double* y, double* out, int64_t n) {
    if (n < 1 || !x || !y || !out) return BODE_E_INVALID_SHAPE;
    int dev = 0;
    if (cudaGetDeviceCount(&dev) != cudaSuccess || dev < 1) {
        cudaGetLastError();
        return BODE_E_NO_DEVICE;
    }
    const double* T = bode::device_powtab();
    double *dx = nullptr, *dy = nullptr, *dz = nullptr;
    if (cudaMalloc(&dx, n * 8) != cudaSuccess || cudaMalloc(&dy, n * 8) != cudaSuccess ||
        cudaMalloc(&dz, n * 8) != cudaSuccess)
        return BODE_E_CUDA;
    cudaMemcpy(dx, x, n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y, n * 8, cudaMemcpyHostToDevice);
    pow_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dx, dy, dz, n, T);
    cudaError_t e = cudaMemcpy(out, dz, n * 8, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dz);
    return e == cudaSuccess ? BODE_OK : BODE_E_CUDA;
}

namespace {
__global__ void exact_math_kernel(const double* __restrict__ x, long long n, int op,
                                  unsigned long long* __restrict__ bad,
                                  unsigned long long* __restrict__ first_bad) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (op == 2 && i + 1 >= n)) return;
    const double v = x[i];
    double got, ref;
    if (op == 2) {  // division: pairs (x[2k], x[2k+1])
        if (i % 2) return;
        const double a = v, b = x[i + 1];
        ref = __ddiv_rn(a, b);
        bool fast;
        got = bode::div_rn_nv<true>(a, b, fast);  // (false only narrows `fast`)
        if (!fast) return;
    } else if (op == 3) {  // the EXACT policy's sqrt_ on every input (fallback included)
        ref = __dsqrt_rn(v);
        got = val(bode::sqrt_(bode::xd(v)));
        if (ref != ref && got != got) return;  // NaN payloads aside
    } else if (op == 4) {  // the EXACT policy's operator/ on every pair (fallback included)
        if (i % 2) return;
        ref = __ddiv_rn(v, x[i + 1]);
        got = val(bode::xd(v) / bode::xd(x[i + 1]));
        if (ref != ref && got != got) return;
    } else {
        if (!bode::in_safe_range(v)) return;
        got = op == 0 ? bode::sqrt_rn_bf(v) : bode::rcp_rn_bf(v);
        ref = op == 0 ? __dsqrt_rn(v) : __drcp_rn(v);
    }
    if (__double_as_longlong(got) != __double_as_longlong(ref)) {
        atomicAdd(bad, 1ull);
        atomicMin(first_bad, (unsigned long long)i);
    }
}
}  // namespace

// Diagnostics: counts the in-range inputs where the branch-free sqrt (op 0)
// or reciprocal (op 1) differs from __dsqrt_rn / __drcp_rn.
extern "C" int bode_selftest_exact_math(const double* x, int64_t n, int32_t op,
                                        int64_t* mismatches, int64_t* first) {
    if (n < 1 || !x || !mismatches) return BODE_E_INVALID_SHAPE;
    int dev = 0;
    if (cudaGetDeviceCount(&dev) != cudaSuccess || dev < 1) {
        cudaGetLastError();
        return BODE_E_NO_DEVICE;
    }
    double* dx = nullptr;
    unsigned long long* db = nullptr;
    if (cudaMalloc(&dx, n * 8) != cudaSuccess || cudaMalloc(&db, 16) != cudaSuccess)
        return BODE_E_CUDA;
    cudaMemcpy(dx, x, n * 8, cudaMemcpyHostToDevice);
    unsigned long long init[2] = {0ull, ~0ull};
    cudaMemcpy(db, init, 16, cudaMemcpyHostToDevice);
    exact_math_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dx, n, op, db, db + 1);
    unsigned long long res[2];
    cudaError_t e = cudaMemcpy(res, db, 16, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(db);
    *mismatches = (int64_t)res[0];
    if (first) *first = res[0] ? (int64_t)res[1] : -1;
    return e == cudaSuccess ? BODE_OK : BODE_E_CUDA;
}
