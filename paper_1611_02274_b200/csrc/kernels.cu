// kernels.cu -- the built-in dispatch table: one entry per (problem, solver,
// arithmetic policy, lane-group width, register cap) compiled for sm_100a.
// The kernel templates themselves are in kernel_entry.cuh.
#include "kernel_entry.cuh"

namespace bode {

long long rkc_table_doubles() { return kRkcTableDoubles; }

const KernelEntry* kernel_table(int* count) {
    static const KernelEntry table[] = {
        // RKCK (nonstiff): Pleiades stages in shared memory, small systems in registers
        // Pleiades: FAST defaults to one lane per system (255 registers, 8 warps/SM);
        // EXACT to the axis split (168 registers, 12 warps/SM) -- the straight-line
        // IEEE sqrt/reciprocal need more registers than one lane can spare
        // (FAST caps measured: 255 -> 5.59e8, 200 -> 4.99e8, 168 -> 4.07e8 system-windows/s)
        make_entry<Pleiades, double, 1, 0, true, 0>(0, 1),
        // (EXACT caps measured: 168 -> 1.91e8, 200 -> 1.88e8, 128 -> 1.79e8 system-windows/s)
        make_entry<Pleiades, xd, 2, 0, true, 168>(0, 0),
        make_entry<Pleiades, double, 2, 0, true, 168>(0, 1),
        make_entry<Pleiades, xd, 1, 0, true, 0>(0, 0),
        BODE_BOTH_ARITH(ExpDecay, 1, 0, false, 2),
        BODE_BOTH_ARITH(Harmonic, 1, 0, false, 3),
        BODE_BOTH_ARITH(Zero<2>, 1, 0, false, 4),
        BODE_BOTH_ARITH(Zero<1>, 1, 0, false, 4),
        BODE_BOTH_ARITH(Riccati, 1, 0, false, 5),
        BODE_BOTH_ARITH(Diag<3>, 1, 0, false, 6),
        BODE_BOTH_ARITH(Const<1>, 1, 0, false, 7),
        BODE_BOTH_ARITH(SinT, 1, 0, false, 8),
        BODE_BOTH_ARITH(Heat<8>, 1, 0, false, 1),
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
        // heatEquation(n) for any other n >= 2: one system per thread block
        make_wide_entry<HeatWide, xd, 0>(1, 0),
        make_wide_entry<HeatWide, double, 0>(1, 1),
        make_wide_entry<HeatWide, xd, 1>(1, 0),
        make_wide_entry<HeatWide, double, 1>(1, 1),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
