"""Summarise an ncu launch list of a generated FT executor run (scripts/ft_profile.py).

Per kernel (k_<loop id>): launches, total / mean duration, share of the profiled
time, DRAM bytes per launch and the achieved DRAM bandwidth (bytes / duration)
against the HBM peak of MEASURED_PEAKS.json; the loop's note from the generated
library tells what it is (mapping, body).

    python scripts/ft_launch_summary.py gpurun_out/r02c/ft_A_launches.csv ft_a [--out md]
"""
import argparse
import collections
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def load(path):
    rows = collections.defaultdict(dict)
    with open(path) as fh:
        lines = [l for l in fh if not l.startswith("==")]
    for r in csv.DictReader(lines):
        name = r["Kernel Name"].split("(")[0]
        rows[int(r["ID"])]["name"] = name
        v = float(r["Metric Value"].replace(",", ""))
        rows[int(r["ID"])][r["Metric Name"]] = v
    return [r for r in rows.values() if "gpu__time_duration.sum" in r]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("app")
    ap.add_argument("--out")
    a = ap.parse_args()
    launches = load(a.csv)
    peak = 6556.8
    try:
        peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:  # noqa: BLE001
        pass
    notes = {}
    try:
        from paper_2002_12115_b200 import generic
        lib = generic.load(a.app)
        notes = {f"k_{l}": lib.loop_notes[l] for l in range(lib.n_loops)}
    except Exception:  # noqa: BLE001
        pass
    agg = collections.OrderedDict()
    for r in launches:
        g = agg.setdefault(r["name"], {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
        g["n"] += 1
        g["ns"] += r["gpu__time_duration.sum"]
        g["rd"] += r.get("dram__bytes_read.sum", 0.0)
        g["wr"] += r.get("dram__bytes_write.sum", 0.0)
    total = sum(g["ns"] for g in agg.values())
    lines = [f"# ncu launch list: {a.app} exact pattern ({len(launches)} launches profiled, "
             f"{total / 1e6:.2f} ms summed kernel time; serialised, cold-cache replay)", "",
             "| kernel | loop | launches | total ms | share | mean us | DRAM MB / launch | "
             "DRAM GB/s | of peak |", "|---|---|---|---|---|---|---|---|---|"]
    for name, g in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        gbs = (g["rd"] + g["wr"]) / g["ns"] if g["ns"] else 0.0
        note = notes.get(name, "")
        lines.append(f"| {name} | {note[:60]} | {g['n']} | {g['ns'] / 1e6:.3f} | "
                     f"{g['ns'] / total:.1%} | {g['ns'] / g['n'] / 1e3:.1f} | "
                     f"{(g['rd'] + g['wr']) / g['n'] / 1e6:.3f} | {gbs:.0f} | {gbs / peak:.1%} |")
    text = "\n".join(lines) + "\n"
    if a.out:
        Path(a.out).write_text(text)
    print(text)


if __name__ == "__main__":
    main()
