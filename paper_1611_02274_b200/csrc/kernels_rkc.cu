// kernels_rkc.cu -- the RKC half of the built-in dispatch table (kernels.cu
// holds the RKCK half and merges all parts): one entry per (problem,
// arithmetic policy, lane-group width, register cap), plus the
// one-system-per-block kernels for heatEquation(n) beyond the padded lane
// groups (wide.cuh).
#include "kernel_entry.cuh"

namespace bode {

const KernelEntry* kernel_table_rkc(int* count) {
    static const KernelEntry table[] = {
        // RKC (moderately stiff)
        // heat64: 8 lanes per system capped at 128 registers (16 warps/SM) is
        // the default -- measured 16% over 4 lanes at 254 registers (8 warps/SM)
        BODE_BOTH_ARITH_R(Heat<64>, 8, 1, false, 1, 128),
        BODE_BOTH_ARITH(Heat<64>, 4, 1, false, 1),
        BODE_BOTH_ARITH_R(Heat<64>, 4, 1, false, 1, 168),
        BODE_BOTH_ARITH_R(Heat<64>, 8, 1, false, 1, 168),
        BODE_BOTH_ARITH_R(Heat<64>, 8, 1, false, 1, 112),
        BODE_BOTH_ARITH_R(Heat<64>, 8, 1, false, 1, 96),
        BODE_BOTH_ARITH_R(Heat<64>, 16, 1, false, 1, 96),
        BODE_BOTH_ARITH_R(Heat<64>, 16, 1, false, 1, 128),
        BODE_BOTH_ARITH(Heat<32>, 4, 1, false, 1),
        BODE_BOTH_ARITH(Heat<16>, 2, 1, false, 1),
        BODE_BOTH_ARITH(Heat<8>, 1, 1, false, 1),
        // expDecay (config 4, controller bound): 80 registers, 24 warps/SM --
        // measured 1.63e8 vs 1.48e8 (128) and 1.23e8 (uncapped, 131) system-windows/s
        BODE_BOTH_ARITH_R(ExpDecay, 1, 1, false, 2, 80),
        BODE_BOTH_ARITH(ExpDecay, 1, 1, false, 2),
        BODE_BOTH_ARITH_R(ExpDecay, 1, 1, false, 2, 128),
        BODE_BOTH_ARITH_R(ExpDecay, 1, 1, false, 2, 96),
        BODE_BOTH_ARITH_R(ExpDecay, 1, 1, false, 2, 64),
        BODE_BOTH_ARITH(Harmonic, 1, 1, false, 3),
        BODE_BOTH_ARITH(Zero<2>, 1, 1, false, 4),
        BODE_BOTH_ARITH(Zero<1>, 1, 1, false, 4),
        BODE_BOTH_ARITH(Diag<3>, 1, 1, false, 6),
        BODE_BOTH_ARITH(Const<1>, 1, 1, false, 7),
        // heatEquation(n) for any n without an exact-size kernel: padded lane
        // groups up to n = 1024 (kernels_pad_a.cu, kernels_pad_b.cu), and for
        // any larger n one system per thread block
        make_wide_entry<HeatWide, xd, 0>(1, 0),
        make_wide_entry<HeatWide, double, 0>(1, 1),
        make_wide_entry<HeatWide, xd, 1>(1, 0),
        make_wide_entry<HeatWide, double, 1>(1, 1),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
