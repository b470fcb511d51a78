// kernels_pad_b.cu -- RKC heatEquation(n) on padded 32-lane groups for
// 224 < n <= 512 (see kernels_pad_a.cu): 8-16 components per lane.
// kernels_pad_c.cu holds 512 < n <= 1024.
#include "kernel_entry.cuh"

#ifndef BODE_PAD_R168
#define BODE_PAD_R168 168  // register cap of the 10-14-component instances (A/B switch)
#endif

namespace bode {

const KernelEntry* kernel_table_pad_b(int* count) {
    static const KernelEntry table[] = {
        BODE_BOTH_ARITH_R(HeatPad<256>, 32, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<288>, 32, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<320>, 32, 1, false, 1, BODE_PAD_R168),
        BODE_BOTH_ARITH_R(HeatPad<384>, 32, 1, false, 1, BODE_PAD_R168),
        make_entry<HeatPad<416>, xd, 32, 1, false, 0>(1, 0),
        make_entry<HeatPad<416>, double, 32, 1, false, BODE_PAD_R168>(1, 1),
        make_entry<HeatPad<448>, xd, 32, 1, false, 0>(1, 0),
        make_entry<HeatPad<448>, double, 32, 1, false, BODE_PAD_R168>(1, 1),
        BODE_BOTH_ARITH_R(HeatPad<512>, 32, 1, false, 1, 0),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
