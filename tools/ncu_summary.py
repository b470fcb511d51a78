#!/usr/bin/env python3
"""Summarise ncu captures for profiles/.

    python tools/ncu_summary.py OUT_PREFIX name=report.ncu-rep:systems [...]
    python tools/ncu_summary.py --launches launches.csv OUT_PREFIX

Writes OUT_PREFIX.md (table) and OUT_PREFIX.json (per kernel: duration, FP64
pipe, issue, occupancy, registers, DRAM bytes per launch and per system, local
spill traffic, warp-state stalls). `systems` is the number of systems the
captured launch integrated (one window), used for the per-system traffic that
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys

RAW = {
    "duration_ns": "gpu__time_duration.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "local_ld_sectors": "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
    "local_st_sectors": "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "thread_inst_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
UNITS = {"dram__bytes_read.sum": 1.0}


def ncu_csv(args):
    r = subprocess.run(["ncu", *args], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1,
            "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9,
            "s": 1e9}.get(unit, 1)


def summarize(report, systems):
    rows = ncu_csv(["-i", report, "--page", "raw", "--csv"])
    hdr, units, vals = rows[0], rows[1], rows[2]
    idx = {h: i for i, h in enumerate(hdr)}
    out = {"kernel": vals[idx["Kernel Name"]], "systems": systems}
    for k, m in RAW.items():
        if m in idx:
            v = vals[idx[m]].replace(",", "")
            try:
                out[k] = float(v) * scale(units[idx[m]])
            except ValueError:
                out[k] = None
    stalls = {}
    for h, i in idx.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i])
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    out["stall_share"] = {k: round(v / tot, 3) for k, v in
                          sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    if out.get("dram_read_bytes") is not None and systems:
        out["dram_bytes_per_system"] = (out["dram_read_bytes"] + out["dram_write_bytes"]) / systems
    if out.get("dram_read_bytes") is not None and out.get("duration_ns"):
        out["dram_GBps"] = (out["dram_read_bytes"] + out["dram_write_bytes"]) / out["duration_ns"]
    if out.get("thread_inst_per_inst") is not None:
        out["warp_execution_efficiency"] = out["thread_inst_per_inst"] / 32.0
    return out


def main():
    if sys.argv[1] == "--launches":
        rows = ncu_csv(["--import", sys.argv[2], "--csv"]) if False else list(
            csv.reader(open(sys.argv[2])))
        hdr = None
        agg = {}
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") != "gpu__time_duration.sum":
                    continue
                name = d["Kernel Name"].split("(")[0]
                t = float(d["Metric Value"].replace(",", "")) * scale(d.get("Metric Unit", ""))
                a = agg.setdefault(name, [0, 0.0])
                a[0] += 1
                a[1] += t
        total = sum(v[1] for v in agg.values()) or 1.0
        with open(sys.argv[3] + ".md", "w") as f:
            f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"| `{k}` | {n} | {t / 1e6:.3f} | {t / total:.1%} |\n")
        print(open(sys.argv[3] + ".md").read())
        return
    prefix = sys.argv[1]
    res = {}
    for spec in sys.argv[2:]:
        name, rest = spec.split("=", 1)
        path, systems = rest.rsplit(":", 1)
        res[name] = summarize(path, int(systems))
    json.dump(res, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write("| capture | kernel | ms | FP64 pipe | warp exec eff | issue | warps | regs | "
                "DRAM B/system | DRAM GB/s | local ld sectors | top stalls |\n"
                "|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for n, r in res.items():
            st = ", ".join(f"{k} {v:.0%}" for k, v in list(r["stall_share"].items())[:4])
            f.write(f"| {n} | `{r['kernel'][:60]}` | {r['duration_ns'] / 1e6:.3f} | "
                    f"{r['fp64_pipe_pct']:.1f}% | {r.get('warp_execution_efficiency', 0):.1%} | "
                    f"{r['issue_active_pct']:.1f}% | "
                    f"{r['warps_active_pct']:.1f}% | {r['registers']:.0f} | "
                    f"{r.get('dram_bytes_per_system', 0):.0f} | {r.get('dram_GBps', 0):.0f} | "
                    f"{r['local_ld_sectors']:.3g} | {st} |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
