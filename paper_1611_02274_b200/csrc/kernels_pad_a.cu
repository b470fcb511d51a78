// kernels_pad_a.cu -- RKC heatEquation(n) on padded lane groups for n <= 224
// without an exact-size kernel (HeatPad<CAP>, problems.cuh: the run-time n
// and 1/dx^2 ride in the kernel's parameter registers, components past n are
// +0.0 and never enter a sum). kernels_pad_b.cu holds the 32-lane groups; the
// dispatcher (host.cu find_entry) takes the smallest capacity >= n.
//
// Capacity = lanes x components per lane. Fewer lanes per system and a
// capacity close to n both pay: against round 2's set (8 components per lane,
// capacities 64/128/256/...) this set measured 1.0x-7x, 1.3x-2.4x over most
// of 64 < n <= 512 (profiles/r02bc_padded_caps.md). Register caps: 9
// components fit 128 (16 warps/SM) under FAST, 168 under EXACT at 8 lanes;
// 10-14 take 168 (12 warps/SM), except FAST at 10 (128 measured 14% faster
// there) and EXACT at 13-14, uncapped (+2-6%; 200 or uncapped costs 5-17%
// elsewhere, r02bo).
#include "kernel_entry.cuh"

#ifndef BODE_PAD_R168
#define BODE_PAD_R168 168  // register cap of the 10-14-component instances (A/B switch)
#endif

namespace bode {

const KernelEntry* kernel_table_pad_a(int* count) {
    static const KernelEntry table[] = {
        BODE_BOTH_ARITH(HeatPad<8>, 1, 1, false, 1),
        BODE_BOTH_ARITH(HeatPad<16>, 2, 1, false, 1),
        BODE_BOTH_ARITH(HeatPad<32>, 4, 1, false, 1),
        BODE_BOTH_ARITH_R(HeatPad<48>, 8, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<64>, 8, 1, false, 1, 128),
        make_entry<HeatPad<72>, xd, 8, 1, false, 168>(1, 0),  // (128: 3-8% slower, r02by)
        make_entry<HeatPad<72>, double, 8, 1, false, 128>(1, 1),
        make_entry<HeatPad<80>, xd, 8, 1, false, BODE_PAD_R168>(1, 0),
        make_entry<HeatPad<80>, double, 8, 1, false, 128>(1, 1),
        BODE_BOTH_ARITH_R(HeatPad<96>, 8, 1, false, 1, BODE_PAD_R168),
        make_entry<HeatPad<104>, xd, 8, 1, false, 0>(1, 0),
        make_entry<HeatPad<104>, double, 8, 1, false, BODE_PAD_R168>(1, 1),
        make_entry<HeatPad<112>, xd, 8, 1, false, 0>(1, 0),
        make_entry<HeatPad<112>, double, 8, 1, false, BODE_PAD_R168>(1, 1),
        BODE_BOTH_ARITH_R(HeatPad<128>, 16, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<144>, 16, 1, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<160>, 16, 1, false, 1, BODE_PAD_R168),
        BODE_BOTH_ARITH_R(HeatPad<192>, 16, 1, false, 1, BODE_PAD_R168),
        make_entry<HeatPad<208>, xd, 16, 1, false, 0>(1, 0),
        make_entry<HeatPad<208>, double, 16, 1, false, BODE_PAD_R168>(1, 1),
        make_entry<HeatPad<224>, xd, 16, 1, false, 0>(1, 0),
        make_entry<HeatPad<224>, double, 16, 1, false, BODE_PAD_R168>(1, 1),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

}  // namespace bode
