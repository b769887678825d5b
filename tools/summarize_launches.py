"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`)
into a per-kernel share table (markdown) for profiles/."""

import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.match(r"void (tl::)?gemm_sm100_kernel<(\d+), \d+, \d+, (\w+), (\w+), (?:tl::)?(?:\(anonymous namespace\)::|<unnamed>::)?(\w+(?:<\d+>)?)>", name)
    if m:
        role = {"EpiLseStats": "K4 fwd", "EpiLseStatsT<0>": "K4 fwd (fp16 store / forward only)",
                "EpiLseStatsT<1>": "K4 fwd (factored store)", "EpiStoreF32": "K5 dW",
                "EpiStoreBF16": "K5 dH", "EpiDSoftmax": "dS recompute"}.get(m.group(5), m.group(5))
        return f"gemm_sm100_kernel<{m.group(2)},..,{m.group(5)}> ({role})"
    return name.split("(")[0][:90]


def main(path: str, title: str = ""):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "nsecond": 1e-6, "second": 1e3, "s": 1e3}.get(unit, 1.0)
        k = short(r["Kernel Name"])
        tot[k] += ms
        cnt[k] += 1
    all_ms = sum(tot.values())
    if title:
        print(title + "\n")
    print("| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / all_ms:.2f}% |")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
