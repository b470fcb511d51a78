#!/usr/bin/env python3
"""Per-source-line warp-stall samples and executed instructions of one ncu capture.

    python tools/ncu_lines.py report.ncu-rep [top]

Reads `ncu --page source --print-source cuda,sass` (the report must have been
captured with -lineinfo and --import-source on) and attributes every SASS row
to the CUDA source line it follows. Prints the top lines by stall samples with
their executed warp instructions and the dominant stall reasons.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    agg = {}
    fname, hdr, cur = None, None, None
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = {k: i for i, k in enumerate(r) if k not in hdr_skip(r, i)}
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:  # a CUDA source row
            cur = (fname, int(r[0]), r[1].strip()[:90])
            continue
        if cur is None:
            continue
        try:
            s = int(r[hdr["# Samples"]] or 0)
            ie = int(r[hdr["Instructions Executed"]] or 0)
        except (ValueError, KeyError):
            continue
        a = agg.setdefault(cur, {"samples": 0, "inst": 0, "stalls": {}})
        a["samples"] += s
        a["inst"] += ie
        for k, i in hdr.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    a["stalls"][k[6:]] = a["stalls"].get(k[6:], 0) + int(r[i] or 0)
                except ValueError:
                    pass
    tot_s = sum(a["samples"] for a in agg.values()) or 1
    tot_i = sum(a["inst"] for a in agg.values()) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        st = sorted(a["stalls"].items(), key=lambda kv: -kv[1])[:3]
        sts = " ".join(f"{n}:{v / max(a['samples'], 1):.0%}" for n, v in st)
        print(f"{a['samples'] / tot_s:6.1%} {a['inst'] / tot_i:6.1%}  {k[0]}:{k[1]:<4} {k[2][:70]:<70} {sts}")


def hdr_skip(row, i):
    # the second "Source" column (SASS text) shares its name with the first
    return {"Source"} if i > 1 and row[i] == "Source" else set()


if __name__ == "__main__":
    main()
