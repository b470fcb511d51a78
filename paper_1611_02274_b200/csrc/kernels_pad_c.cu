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
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
