// repack.cu -- cost-aware re-packing of a device-resident batch.
//
// A warp advances its lane groups in lockstep, so a window costs each warp
// its slowest system. When per-system cost varies a lot inside warps -- the
// RKC stage count grows with sqrt(h * sigma), so a stiffness-varied batch in
// natural order (BASELINE config 4) runs at ~0.3 lockstep efficiency --
// sorting the systems by the cost they just showed (the window's RHS
// evaluations, in the per-system stats) puts similar systems in the same
// warps. Every system is integrated independently and deterministically
// (batch_driver.hpp:16-21), so the results are bitwise the same in any order;
// only the position of a system in the arrays changes, tracked by `order`
// (position -> original index) and undone by bode_unpack.
//
// Sorting is CUB's device radix sort (32-bit saturated keys, stable); the
// permutation is a gather into scratch plus a device copy back, so the caller's
// buffers keep their addresses.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <mutex>
#include <string>

#include "../../include/bode.h"
#include "dispatch.h"

namespace {

using bode::DevStats;

// Scratch comes from the stream-ordered allocator on the call's own stream
// (cudaMallocAsync / cudaFreeAsync), so concurrent calls on different streams
// -- or a user call next to bode_outer_loop's internal stream -- never share
// it. The device's default pool keeps freed blocks (release threshold raised
// once per device), so a warm call does not reach the driver allocator.
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

int scratch(int dev, size_t bytes, cudaStream_t s, Scratch* out) {
    static std::once_flag once[64];
    if (dev < 0 || dev >= 64) return BODE_E_UNSUPPORTED;
    std::call_once(once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
    if (cudaMallocAsync(&out->p, bytes, s) != cudaSuccess) {
        out->p = nullptr;
        return BODE_E_CUDA;
    }
    out->s = s;
    return BODE_OK;
}

__global__ void cost_keys(const DevStats* __restrict__ st, long long num,
                          unsigned* __restrict__ key, unsigned* __restrict__ idx) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= num) return;
    const long long c = st[i].rhs_evals;
    key[i] = c < 0 ? 0u : c > 0xffffffffll ? 0xffffffffu : (unsigned)c;
    idx[i] = (unsigned)i;
}

// key = |g_row[i]| rounded to float: for non-negative floats the bit pattern
// orders like the value (NaN sorts last)
__global__ void param_keys(const double* __restrict__ g_row, long long num,
                           unsigned* __restrict__ key, unsigned* __restrict__ idx) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= num) return;
    key[i] = __float_as_uint(fabsf(__double2float_rn(g_row[i])));
    idx[i] = (unsigned)i;
}

// dst[j*num + p] = src[j*num + from[p]] (SoA gather, coalesced writes)
__global__ void gather_soa(const double* __restrict__ src, double* __restrict__ dst, int rows,
                           long long num, const unsigned* __restrict__ from) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= num) return;
    const long long f = from[p];
    for (int j = 0; j < rows; ++j) dst[j * num + p] = src[j * num + f];
}

// dst[j*num + to[p]] = src[j*num + p] (SoA scatter)
__global__ void scatter_soa(const double* __restrict__ src, double* __restrict__ dst, int rows,
                            long long num, const long long* __restrict__ to) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= num) return;
    const long long t = to[p];
    for (int j = 0; j < rows; ++j) dst[j * num + t] = src[j * num + p];
}

__global__ void gather_stats_order(const DevStats* __restrict__ st, DevStats* __restrict__ st2,
                                   const long long* __restrict__ ord, long long* __restrict__ ord2,
                                   long long num, const unsigned* __restrict__ from) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= num) return;
    const long long f = from[p];
    if (st) st2[p] = st[f];
    ord2[p] = ord[f];
}

__global__ void scatter_stats(const DevStats* __restrict__ st, DevStats* __restrict__ st2,
                              long long num, const long long* __restrict__ to) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= num) return;
    st2[to[p]] = st[p];
}

__global__ void identity_order(long long* __restrict__ ord, long long num) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < num) ord[p] = p;
}

// sum over systems of cost, and of the cost of each system's warp group's
// slowest member (groups of `group` consecutive systems, group | 32)
__global__ void lockstep_sums(const DevStats* __restrict__ st, long long num, int group,
                              unsigned long long* __restrict__ sums) {
    // grid-stride over warp-aligned positions (the stride is a multiple of 32,
    // so a lane group never straddles two iterations), shuffle reductions per
    // warp, then one atomic pair per block: a few thousand atomics instead of
    // one pair per warp
    __shared__ unsigned long long part[2][32];
    unsigned long long s = 0ull, w = 0ull;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x % 32 < num;
         i += stride) {
        const bool valid = i < num;
        const long long c0 = valid ? st[i].rhs_evals : 0;
        const unsigned long long c = c0 > 0 ? (unsigned long long)c0 : 0ull;
        unsigned long long m = c;
        for (int o = group / 2; o > 0; o /= 2) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
            m = t > m ? t : m;
        }
        s += c;
        w += valid ? m : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o /= 2) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        w += __shfl_xor_sync(0xffffffffu, w, o);
    }
    const int warp = threadIdx.x / 32, nwarps = blockDim.x / 32;
    if ((threadIdx.x & 31) == 0) {
        part[0][warp] = s;
        part[1][warp] = w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long bs = 0ull, bw = 0ull;
        for (int k = 0; k < nwarps; ++k) {
            bs += part[0][k];
            bw += part[1][k];
        }
        atomicAdd(&sums[0], bs);
        atomicAdd(&sums[1], bw);
    }
}

// Publishes the two sums into pinned host memory from the device (UVA), so
// the read-back needs no copy engine: a D2H memcpy here would queue behind
// the outer loop's multi-gigabyte snapshot copy on the same engine and
// serialise it with the next window's kernel.
__global__ void publish_sums(const unsigned long long* __restrict__ d,
                             volatile unsigned long long* h) {
    h[0] = d[0];
    h[1] = d[1];
    __threadfence_system();
}

inline unsigned blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

int cuda_fail(cudaError_t e) {
    (void)e;
    return BODE_E_CUDA;
}

#define RP_CUDA(call)                                      \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_);       \
    } while (0)

}  // namespace

namespace bode {

// Sorts the systems by a key and permutes y, g, stats (may be null) and order
// accordingly: the cost each system just showed (stats[i].rhs_evals) when
// param_row < 0, else the magnitude of parameter row param_row (a stiffness
// proxy such as expDecay's g0, known before the first window). All pointers
// are device pointers on the current device.
int repack_by(int N, int P, long long num, double* y, double* g, DevStats* st, long long* order,
              int param_row, cudaStream_t s) {
    if (num < 2 || order == nullptr) return BODE_OK;
    if (param_row < 0 ? st == nullptr : (param_row >= P || g == nullptr))
        return BODE_E_INVALID_SHAPE;
    int dev = 0;
    RP_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return BODE_E_UNSUPPORTED;
    size_t sort_bytes = 0;
    RP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (unsigned*)nullptr,
                                            (unsigned*)nullptr, (unsigned*)nullptr,
                                            (unsigned*)nullptr, (int)num, 0, 32, s));
    const size_t n = (size_t)num;
    const int rows = N > P ? N : P;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t bytes = 4 * al(n * sizeof(unsigned)) + al(sort_bytes) +
                         al(n * rows * sizeof(double)) + al(n * sizeof(DevStats)) +
                         al(n * sizeof(long long));
    Scratch sc;
    if (scratch(dev, bytes, s, &sc) != BODE_OK) return BODE_E_CUDA;
    char* c = static_cast<char*>(sc.p);
    unsigned* key = reinterpret_cast<unsigned*>(c);
    c += al(n * sizeof(unsigned));
    unsigned* key2 = reinterpret_cast<unsigned*>(c);
    c += al(n * sizeof(unsigned));
    unsigned* idx = reinterpret_cast<unsigned*>(c);
    c += al(n * sizeof(unsigned));
    unsigned* from = reinterpret_cast<unsigned*>(c);
    c += al(n * sizeof(unsigned));
    void* tmp = c;
    c += al(sort_bytes);
    double* buf = reinterpret_cast<double*>(c);
    c += al(n * rows * sizeof(double));
    DevStats* st2 = reinterpret_cast<DevStats*>(c);
    c += al(n * sizeof(DevStats));
    long long* ord2 = reinterpret_cast<long long*>(c);

    if (param_row < 0)
        cost_keys<<<blocks(num, 256), 256, 0, s>>>(st, num, key, idx);
    else
        param_keys<<<blocks(num, 256), 256, 0, s>>>(g + (size_t)param_row * n, num, key, idx);
    RP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, key, key2, idx, from, (int)num, 0,
                                            32, s));
    gather_soa<<<blocks(num, 256), 256, 0, s>>>(y, buf, N, num, from);
    RP_CUDA(cudaMemcpyAsync(y, buf, n * N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (P > 0 && g != nullptr) {
        gather_soa<<<blocks(num, 256), 256, 0, s>>>(g, buf, P, num, from);
        RP_CUDA(cudaMemcpyAsync(g, buf, n * P * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    gather_stats_order<<<blocks(num, 256), 256, 0, s>>>(st, st2, order, ord2, num, from);
    if (st != nullptr)
        RP_CUDA(cudaMemcpyAsync(st, st2, n * sizeof(DevStats), cudaMemcpyDeviceToDevice, s));
    RP_CUDA(cudaMemcpyAsync(order, ord2, n * sizeof(long long), cudaMemcpyDeviceToDevice, s));
    RP_CUDA(cudaGetLastError());
    return BODE_OK;
}

int repack_by_cost(int N, int P, long long num, double* y, double* g, DevStats* st,
                   long long* order, cudaStream_t s) {
    return repack_by(N, P, num, y, g, st, order, -1, s);
}

// Scatters y (and g, stats) back to original positions and resets order.
// With y_out != nullptr only y is scattered, into y_out (a snapshot), and
// nothing else changes.
int unpack(int N, int P, long long num, double* y, double* g, DevStats* st, long long* order,
           double* y_out, cudaStream_t s) {
    if (num < 1 || order == nullptr) return BODE_OK;
    if (y_out != nullptr) {
        scatter_soa<<<blocks(num, 256), 256, 0, s>>>(y, y_out, N, num, order);
        RP_CUDA(cudaGetLastError());
        return BODE_OK;
    }
    int dev = 0;
    RP_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return BODE_E_UNSUPPORTED;
    const size_t n = (size_t)num;
    const int rows = N > P ? N : P;
    const size_t bytes = ((n * rows * sizeof(double) + 255) & ~size_t(255)) + n * sizeof(DevStats);
    Scratch sc;
    if (scratch(dev, bytes, s, &sc) != BODE_OK) return BODE_E_CUDA;
    void* base = sc.p;
    double* buf = static_cast<double*>(base);
    DevStats* st2 = reinterpret_cast<DevStats*>(static_cast<char*>(base) +
                                                ((n * rows * sizeof(double) + 255) & ~size_t(255)));
    scatter_soa<<<blocks(num, 256), 256, 0, s>>>(y, buf, N, num, order);
    RP_CUDA(cudaMemcpyAsync(y, buf, n * N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (P > 0 && g != nullptr) {
        scatter_soa<<<blocks(num, 256), 256, 0, s>>>(g, buf, P, num, order);
        RP_CUDA(cudaMemcpyAsync(g, buf, n * P * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    if (st != nullptr) {
        scatter_stats<<<blocks(num, 256), 256, 0, s>>>(st, st2, num, order);
        RP_CUDA(cudaMemcpyAsync(st, st2, n * sizeof(DevStats), cudaMemcpyDeviceToDevice, s));
    }
    identity_order<<<blocks(num, 256), 256, 0, s>>>(order, num);
    RP_CUDA(cudaGetLastError());
    return BODE_OK;
}

int init_order(long long* order, long long num, cudaStream_t s) {
    identity_order<<<blocks(num, 256), 256, 0, s>>>(order, num);
    RP_CUDA(cudaGetLastError());
    return BODE_OK;
}

// Lockstep efficiency of the stats' costs for warps of `group` systems:
// sum(cost) / sum(group max * group size). Synchronises the stream.
int lockstep_efficiency(const DevStats* st, long long num, int group, double* eff,
                        cudaStream_t s) {
    // per-device device/pinned-host counter pair, allocated once
    static std::mutex m;
    static unsigned long long* dsum[64] = {nullptr};
    static unsigned long long* hsum[64] = {nullptr};
    static unsigned long long* hsum_dev[64] = {nullptr};  // its device alias
    int dev = 0;
    RP_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return BODE_E_UNSUPPORTED;
    std::lock_guard<std::mutex> lock(m);
    if (dsum[dev] == nullptr) {
        RP_CUDA(cudaMalloc(&dsum[dev], 2 * sizeof(unsigned long long)));
        RP_CUDA(cudaHostAlloc(&hsum[dev], 2 * sizeof(unsigned long long),
                              cudaHostAllocMapped | cudaHostAllocPortable));
        RP_CUDA(cudaHostGetDevicePointer((void**)&hsum_dev[dev], hsum[dev], 0));
    }
    RP_CUDA(cudaMemsetAsync(dsum[dev], 0, 2 * sizeof(unsigned long long), s));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<long long>(blocks(num, 256), 8ll * sms);
    lockstep_sums<<<grid, 256, 0, s>>>(st, num, group, dsum[dev]);
    publish_sums<<<1, 1, 0, s>>>(dsum[dev], hsum_dev[dev]);
    RP_CUDA(cudaGetLastError());
    RP_CUDA(cudaStreamSynchronize(s));
    *eff = hsum[dev][1] ? (double)hsum[dev][0] / (double)hsum[dev][1] : 1.0;
    return BODE_OK;
}

}  // namespace bode
