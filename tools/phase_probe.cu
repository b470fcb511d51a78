// phase_probe.cu -- where the RKC heat64 kernel's time goes, phase by phase.
// Builds the production kernel with BODE_PHASE_TIMING (clock64() deltas per
// rkc_system phase, rkc.cuh) and integrates 2^20 systems over two windows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -Ipaper_1611_02274_b200/csrc -DBODE_PHASE_TIMING tools/phase_probe.cu -o phase_probe
// The instrumentation perturbs scheduling a little; read the shares, not ms.
#include <cmath>
#include <cstdio>
#include <vector>

#include "kernel_entry.cuh"

using namespace bode;

int main() {
    const long long num = 1 << 20;
    const int N = 64;
    std::vector<double> y(num * N);
    for (long long i = 0; i < num; ++i)
        for (int j = 0; j < N; ++j) {
            const double x = (j + 1.0) / (N + 1.0);
            y[i + num * j] = 4 * x * (1 - x) * (1 + 0.01 * std::sin(i * 0.1 + j));
        }
    double* dy;
    DevStats* st;
    cudaMalloc(&dy, y.size() * 8);
    cudaMalloc(&st, num * sizeof(DevStats));
    cudaMemcpy(dy, y.data(), y.size() * 8, cudaMemcpyHostToDevice);
    unsigned long long* ph;
    cudaMalloc(&ph, 5 * 8);
    cudaMemcpyToSymbol(g_phase, &ph, sizeof(ph));
    const KernelEntry e = make_entry<Heat<64>, xd, 8, 1, false, 128>(1, 0);
    double* tab;
    cudaMalloc(&tab, kRkcTableDoubles * 8);
    e.build_rkc_table(tab, 2.0 / 13.0, 0);
    const DevTol tol{1e-10, 1e-10, 1e-6, 2.22e-16, 1e-30, 0.9, 0.1, 1.89e-4, -0.2, -0.25, 1e-20,
                     2.0 / 13.0, nullptr, tab, 8, 0};
    const int block = 128;
    const long long grid = (num * 8 + block - 1) / block;
    const size_t smem = (size_t)e.smem_per_thread * block;
    e.prepare(e.fn, 0, (int)smem);
    const char* names[5] = {"power method", "initial step", "stage loop", "f_trial+error norm",
                            "controller"};
    for (int w = 0; w < 2; ++w) {
        cudaMemset(ph, 0, 40);
        e.launch(e.fn, dim3(grid), dim3(block), smem, 0, nullptr, dy, st, num, 0.1 * w,
                 0.1 * (w + 1), tol, 0);
        unsigned long long h[5];
        cudaMemcpy(h, ph, 40, cudaMemcpyDeviceToHost);
        double tot = 0;
        for (int k = 0; k < 5; ++k) tot += h[k];
        std::printf("window %d (%s)\n", w, cudaGetErrorString(cudaGetLastError()));
        for (int k = 0; k < 5; ++k) std::printf("  %-20s %5.1f%%\n", names[k], 100.0 * h[k] / tot);
    }
    return 0;
}
