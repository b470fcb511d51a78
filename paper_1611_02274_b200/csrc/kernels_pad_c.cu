// kernels_pad_c.cu -- RKC heatEquation(n) on padded 32-lane groups for
// 512 < n <= 1024 (see kernels_pad_a.cu): 18-32 components per lane, every
// 64 components, uncapped registers (EXACT spills at some capacities but
// still beats one system per block, 1.4-2.2x, r02al). Against capacities
// 768 and 1024 alone the 64-step set measured 1.1-1.7x (r02ci, r02cj).
#include "kernel_entry.cuh"

namespace bode {

const KernelEntry* kernel_table_pad_c(int* count) {
    static const KernelEntry table[] = {
        BODE_BOTH_ARITH_R(HeatPad<576>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<640>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<704>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<768>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<832>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<896>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<960>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<1024>, 32, 1, false, 1, 0),
        // FAST only past 1024: 1.6-1.8x over one system per block at n = 1100 /
        // 1250, while EXACT (heavier spills) measured 1.04x / 0.92x (r02cm)
        make_entry<HeatPad<1152>, double, 32, 1, false, 0>(1, 1),
        make_entry<HeatPad<1280>, double, 32, 1, false, 0>(1, 1),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
