// fp64_latency.cu -- dependent-chain latencies on this device (one warp,
// clock64 around 1024 dependent operations), for the serial phases of the RKC
// driver (the error-norm sum chain, the controller's division/cbrt chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>

#include <cuda_runtime.h>

constexpr int kN = 1024;

__global__ void chains(double* out, long long* cyc, double a, double b) {
    double x = threadIdx.x * 1e-3 + 1.0;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < kN; ++i) x = __dadd_rn(x, a);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < kN; ++i) x = __dmul_rn(x, b);
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DFMA chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < kN; ++i) x = fma(x, b, a);
    t1 = clock64();
    cyc[2] = t1 - t0;
    // shuffle + DADD chain (the lane hand-off of a sequential sum)
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < kN; ++i) x = __dadd_rn(__shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31), a);
    t1 = clock64();
    cyc[3] = t1 - t0;
    // IEEE division chain (intrinsic, fast path)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < kN / 8; ++i) x = __ddiv_rn(x, b) + a;
    t1 = clock64();
    cyc[4] = t1 - t0;
    // shared-memory load -> DADD chain (address depends on the previous value)
    __shared__ double sm[64];
    sm[threadIdx.x] = a;
    sm[threadIdx.x + 32] = a;
    __syncwarp();
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < kN / 8; ++i) x = __dadd_rn(x, sm[(threadIdx.x + (x > 1e300)) & 63]);
    t1 = clock64();
    cyc[5] = t1 - t0;
    out[threadIdx.x] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    for (int rep = 0; rep < 2; ++rep) chains<<<1, 32>>>(out, cyc, 1e-17, 0.999999);
    cudaDeviceSynchronize();
    const char* name[6] = {"DADD", "DMUL", "DFMA", "SHFL+DADD", "DDIV(+DADD)", "LDS+DADD"};
    const int n[6] = {kN, kN, kN, kN, kN / 8, kN / 8};
    printf("{");
    for (int k = 0; k < 6; ++k)
        printf("%s\"%s\": %.2f", k ? ", " : "", name[k], double(cyc[k]) / n[k]);
    printf("}\n");
    return 0;
}
