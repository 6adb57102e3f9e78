"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel.

    python scripts/launch_summary.py gpurun_out/<tag>/launches.csv [--out profiles/x.md]
"""
import argparse
import csv
import re
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out")
    args = ap.parse_args()
    lines = open(args.csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("unnamed>::", "")
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        agg[name][0] += 1
        agg[name][1] += ns
    total = sum(v[1] for v in agg.values())
    out = [f"# launch list: {args.csv}", "",
           "ncu `gpu__time_duration.sum`, cold-cache serialised launches: compare shares, "
           "not absolutes.", "",
           "| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name}` | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {ns / total:.1%} |")
    text = "\n".join(out)
    if args.out:
        open(args.out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
