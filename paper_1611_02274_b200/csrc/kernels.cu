// kernels.cu -- the built-in dispatch table: one entry per (problem, solver,
// arithmetic policy, lane-group width, register cap) compiled for sm_100a.
// The kernel templates themselves are in kernel_entry.cuh.
#include <vector>

#include "kernel_entry.cuh"

namespace bode {

long long rkc_table_doubles() { return kRkcTableDoubles; }

// kernels_rkc.cu: the RKC entries and the one-system-per-block heat kernels
// (a second translation unit, so the two halves compile in parallel)
const KernelEntry* kernel_table_rkc(int* count);
// kernels_pad_{a,b,c}.cu: RKC heatEquation(n) on padded lane groups
const KernelEntry* kernel_table_pad_a(int* count);
const KernelEntry* kernel_table_pad_b(int* count);
const KernelEntry* kernel_table_pad_c(int* count);

static const KernelEntry* kernel_table_rkck(int* count) {
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
        // heatEquation(n), n <= 64 without an exact-size kernel (RKCK): padded groups
        BODE_BOTH_ARITH(HeatPad<16>, 2, 0, false, 1),
        // (32 and 48: 1.3-2.2x over padding to 64 at n = 17-48, r02bl)
        BODE_BOTH_ARITH_R(HeatPad<32>, 4, 0, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<48>, 8, 0, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<64>, 8, 0, false, 1, 128),
        // n in (64, 768]: 1.4-4.2x over one system per block (r02cc, r02cd,
        // r02cg); 512 and 768 keep the stages in shared memory, 128 and 256 in
        // registers (stages in shared memory measured 2-3% slower there)
        BODE_BOTH_ARITH_R(HeatPad<128>, 16, 0, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<256>, 32, 0, false, 1, 128),
        BODE_BOTH_ARITH_R(HeatPad<512>, 32, 0, true, 1, 0),
        // 768: 1.4x / 2.1x (EXACT / FAST) at n = 600; a 1024 capacity lost to
        // the block kernel under EXACT (0.80x at n = 1000, r02cg)
        BODE_BOTH_ARITH_R(HeatPad<768>, 32, 0, true, 1, 0),
    };
    *count = (int)(sizeof(table) / sizeof(table[0]));
    return table;
}

const KernelEntry* kernel_table(int* count) {
    static const std::vector<KernelEntry> all = [] {
        std::vector<KernelEntry> v;
        int n = 0;
        const KernelEntry* a = kernel_table_rkck(&n);
        v.insert(v.end(), a, a + n);
        for (auto part : {kernel_table_rkc, kernel_table_pad_a, kernel_table_pad_b,
                          kernel_table_pad_c}) {
            const KernelEntry* b = part(&n);
            v.insert(v.end(), b, b + n);
        }
        return v;
    }();
    *count = (int)all.size();
    return all.data();
}

}  // namespace bode
