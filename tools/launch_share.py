"""Per-kernel share of an ncu launch list (``--metrics gpu__time_duration.sum --csv``).

    python tools/launch_share.py gpurun_out/launches.csv > profiles/<round>/launch_share.md

ncu times are cold-cache and serialised: compare each kernel's SHARE of
the step with bench.py's CUDA-event split, not the absolute times.
"""

import collections
import csv
import sys


def main(path: str) -> None:
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(lines[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        a = agg[r["Kernel Name"]]
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"launch list: `{path}` ({sum(v[0] for v in agg.values())} launches)\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {t / n:.1f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
