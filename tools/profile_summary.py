"""Turn an `ncu --set full` capture of tools/ncu_targets.py (one ~1-chunk C2
GRPO step) into the committed evidence under profiles/:

    python tools/profile_summary.py gpurun_out/prof.ncu-rep profiles/<round>

writes <prefix>_ncu_full_raw_metrics.csv (selected raw metrics per launch),
<prefix>_ncu_full_summary.md (table) and <prefix>_gemm_traffic.json (DRAM
bytes of the first fwd / dH / dW launch = one full chunk), which bench.py
reads for roofline.traffic."""

import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size",
]
ROLE = {"EpiLseStats": "gemm_fwd", "EpiStoreBF16": "gemm_dh", "EpiStoreF32": "gemm_dw",
        "EpiDSoftmax": "gemm_ds"}


def role(name):
    for k, v in ROLE.items():
        if "gemm_sm100" in name and k in name:
            return v
    for k in ("dsoftmax", "gather_rows", "gather_anchor", "fixup_rows", "scale_rows", "pack_scatter", "pack_scan", "group_adv",
              "loss_unit_kernel<true>", "loss_unit_kernel<false>", "loss_finalize"):
        if k in name:
            return k
    return name.split("(")[0][-40:]


def main(rep, prefix, chunk_rows=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    keep = ["ID", "Kernel Name"] + [m for m in METRICS if m in hdr]
    idx = [hdr.index(k) for k in keep]
    with open(prefix + "_ncu_full_raw_metrics.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(keep)
        w.writerow([units[i] for i in idx])
        for r in data:
            w.writerow([r[i] for i in idx])
    col = {k: hdr.index(k) for k in keep}

    def val(r, m):
        try:
            return float(r[col[m]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")

    lines = ["| # | kernel | ms | SM GHz | DRAM rd GB | DRAM wr GB | DRAM % | tensor % | SM % | warp-instr |",
             "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
    per_chunk = {}
    for r in data:
        k = role(r[col["Kernel Name"]])
        ms = val(r, "gpu__time_duration.sum")
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        lines.append(f"| {r[col['ID']]} | `{k}` | {ms:.3f} | {val(r, 'sm__cycles_elapsed.avg.per_second'):.2f} | "
                     f"{rd:.2f} | {wr:.2f} | {val(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{val(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{val(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{val(r, 'smsp__inst_executed.sum'):.3g} |")
        if k.startswith("gemm") or k == "dsoftmax":
            per_chunk.setdefault(k, {"dram_read_GB": rd, "dram_write_GB": wr, "ms": ms})
    with open(prefix + "_ncu_full_summary.md", "w") as f:
        f.write(f"# `ncu --set full --clock-control none` of tools/ncu_targets.py ({rep.split('/')[-1]})\n\n"
                "One ~1-chunk C2 GRPO step (chunk = first launch of each kind; the second, smaller "
                "launches are the remainder chunk).  ncu replays each kernel in isolation with caches "
                "flushed: compare shares and bytes, not absolute times.\n\n")
        f.write("\n".join(lines) + "\n")
    tj = {"source": prefix + "_ncu_full_raw_metrics.csv (ncu --set full, tools/ncu_targets.py)",
          "chunk_rows": int(chunk_rows) if chunk_rows else 37888, "H": 3584, "V": 152064,
          "per_chunk": per_chunk}
    with open(prefix + "_gemm_traffic.json", "w") as f:
        json.dump(tj, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
