// kernels_pad_b.cu -- RKC heatEquation(n) on padded 32-lane groups for
// 224 < n <= 1024 (see kernels_pad_a.cu). 8-16 components per lane; 768 and
// 1024 spill under EXACT but still beat one system per block (2.2x at n =
// 600, 1.4x at n = 1000, r02al).
#include "kernel_entry.cuh"

namespace bode {

const KernelEntry* kernel_table_pad_b(int* count) {
    static const KernelEntry table[] = {
        BODE_BOTH_ARITH_R(HeatPad<256>, 32, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<288>, 32, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<320>, 32, 1, false, 1, 168),
        BODE_BOTH_ARITH_R(HeatPad<384>, 32, 1, false, 1, 168),
        BODE_BOTH_ARITH_R(HeatPad<416>, 32, 1, false, 1, 168),
        BODE_BOTH_ARITH_R(HeatPad<448>, 32, 1, false, 1, 168),
        BODE_BOTH_ARITH_R(HeatPad<512>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<768>, 32, 1, false, 1, 0),
        BODE_BOTH_ARITH_R(HeatPad<1024>, 32, 1, false, 1, 0),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
