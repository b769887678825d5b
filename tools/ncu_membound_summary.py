"""Summarise an `ncu --set full` capture of tools/ncu_membound.py (K1 / K2 /
K3 at a full config shape) into markdown: per kernel launch its duration,
DRAM bytes and throughput, instructions, issue rate and top stall reasons.

    python tools/ncu_membound_summary.py report.ncu-rep > profiles/<prefix>_ncu_membound_summary.md
"""

import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__registers_per_thread"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    c = {k: i for i, k in enumerate(hdr)}
    # raw-page units vary with magnitude: normalise to us and MB
    to_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    to_mb = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    stall = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
             and k.endswith("_per_issue_active.ratio")]
    print(f"# `ncu --set full` of the memory-bound kernels ({rep.split('/')[-1]}, tools/ncu_membound.py)\n")
    print("Each operation ran twice; both launches are listed (caches flushed by ncu before each replay). "
          "DRAM write bytes undercount stores that are still dirty in the 126 MB L2 at kernel end.\n")
    print("| # | kernel | grid | regs | µs | DRAM rd MB | DRAM wr MB | DRAM % | warp-instr | issue/cycle | warps active % | top stalls (cycles per issue) |")
    print("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|")

    def f(r, k, scale=1.0):
        try:
            v = float(r[c[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
        u = units[c[k]]
        return v * to_us.get(u, to_mb.get(u, scale))

    for r in data:
        name = r[c["Kernel Name"]].split("(")[0].replace("tl::", "").replace("<unnamed>::", "")
        st = sorted(((f(r, k), k.split("stalled_")[1].split("_per_issue")[0]) for k in stall),
                    reverse=True)[:3]
        print(f"| {r[c['ID']]} | `{name[:40]}` | {f(r, 'launch__grid_size'):.0f} | "
              f"{f(r, 'launch__registers_per_thread'):.0f} | {f(r, 'gpu__time_duration.sum'):.1f} | "
              f"{f(r, 'dram__bytes_read.sum'):.1f} | {f(r, 'dram__bytes_write.sum'):.1f} | "
              f"{f(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{f(r, 'smsp__inst_executed.sum'):.3g} | {f(r, 'smsp__issue_active.avg.per_cycle_active'):.2f} | "
              f"{f(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              + ", ".join(f"{n} {v:.1f}" for v, n in st) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
