"""profiles/<prefix>_bench_cN.json.log -> profiles/<prefix>_configs.md (one row per BASELINE config)."""

import json
import sys
from pathlib import Path

PROF = Path(__file__).resolve().parents[1] / "profiles"


def main(prefix: str):
    rows = []
    for c in ["c1", "c2", "c3", "c4", "c5"]:
        p = PROF / f"{prefix}_bench_{c}.json.log"
        if not p.exists():
            continue
        d = json.loads(p.read_text().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        cb = d.get("cpu_baseline") or {}
        nan = float("nan")
        rows.append(f"| {c} | {d['config']['workload']} | {d['config']['tokens_per_step']:,} | "
                    f"{d['config']['action_tokens_per_step']:,} | {d.get('impl_config', {}).get('micro_batches', d['config'].get('micro_batches', 1))} | "
                    f"{d['ms_per_step']:.1f} | {d['value']:,.0f} | {e.get('value', nan):,.0f} | "
                    f"{r.get('frac', nan):.3f} | {r.get('step_frac', nan):.3f} | "
                    f"{d['clocks'].get('sm_mhz')} | {cb.get('value', nan):.1f} |")
    hdr = ("| config | workload | tokens/step | action tokens | micro-batches | ms/step | tokens/s | "
           "e2e tokens/s | GEMM frac | step frac | SM MHz | CPU ref tokens/s |\n"
           "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
    text = (f"# {prefix} bench lines for every BASELINE.json config (1 x B200, `python bench.py --config cN`)\n\n"
            "Fraction = algorithmic 6*T_act*H*V over the GEMMs' event time (frac) / over the whole step "
            "(step frac), against MEASURED_PEAKS.json bf16_tflops_sustained.  C3/C4 hold more activations "
            "than HBM, so each step runs as micro-batches of whole groups (global normalisers, dW accumulated, "
            "reports combined).  C3 is run with --no-e2e.  C1 (H 896, V 32k, 18.6 k action rows: one small chunk) is launch- and tail-bound.  Boxes "
            "differ by ~3 %.  Raw JSON lines: " + f"{prefix}_bench_cN.json.log.\n\n" + hdr + "\n" +
            "\n".join(rows) + "\n")
    (PROF / f"{prefix}_configs.md").write_text(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1f")
