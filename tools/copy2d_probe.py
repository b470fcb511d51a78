#!/usr/bin/env python3
"""PCIe cost of the host-pointer pipeline's pitched copies against the batch
size: 28 SoA rows of `num` doubles in pinned host memory, copied in 32 column
chunks (cudaMemcpy2DAsync, host pitch num*8, device pitch chunk*8) H2D and
back D2H, each direction alone (CUDA events). Shows how the row alignment of
the caller's array affects the DMA.

    python tools/copy2d_probe.py
"""
import json

import torch
from cuda.bindings import runtime as rt

ROWS, NCH = 28, 32


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    assert err == rt.cudaError_t.cudaSuccess, err


def run(num, per_row=False, reps=3, align=1):
    h = torch.zeros(num * ROWS, dtype=torch.float64).pin_memory()
    d = torch.empty(num * ROWS, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    cb, rem = divmod(num, NCH)
    chunks, off = [], 0
    for c in range(NCH):
        nk = cb + (1 if c < rem else 0)
        if align > 1:  # chunk widths rounded to `align` systems, the last takes the rest
            nk = num - off if c == NCH - 1 else (cb // align) * align
        chunks.append((off, nk))
        off += nk
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def go(kind):
        for off, nk in chunks:
            hp = h.data_ptr() + off * 8
            dp = d.data_ptr() + off * ROWS * 8
            if per_row:
                for r in range(ROWS):
                    a, b = (dp + r * nk * 8, hp + r * num * 8)
                    ck(rt.cudaMemcpyAsync(*(a, b) if kind == H2D else (b, a), nk * 8, kind,
                                          s.cuda_stream))
            elif kind == H2D:
                ck(rt.cudaMemcpy2DAsync(dp, nk * 8, hp, num * 8, nk * 8, ROWS, kind, s.cuda_stream))
            else:
                ck(rt.cudaMemcpy2DAsync(hp, num * 8, dp, nk * 8, nk * 8, ROWS, kind, s.cuda_stream))

    out = {}
    for name, kind in (("h2d", H2D), ("d2h", D2H)):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            go(kind)
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name + "_ms"] = round(best, 2)
        out[name + "_GBps"] = round(num * ROWS * 8 / best / 1e6, 1)
    return out


def main():
    for num in (1 << 24, (1 << 24) - 32, 16760017, 16760832):
        for align in (1, 32, 512):
            r = run(num, False, align=align)
            r.update({"num": num, "host_pitch_mod_4096": num * 8 % 4096, "chunk_align": align})
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
