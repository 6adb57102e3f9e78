"""Summarise ncu reports (--page raw) into profiles/: key metrics per kernel launch.

    python scripts/ncu_summary.py gpurun_out/<tag>/<name>.ncu-rep [--out profiles/<file>.md]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--out")
    ap.add_argument("--bytes-per-launch", type=float, default=None,
                    help="algorithmic bytes per launch (for traffic ratio)")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary: {args.report}", ""]
    out = []
    for r in rows[2:]:
        name = r[idx["Kernel Name"]] if "Kernel Name" in idx else "?"
        rec = {"kernel": name}
        lines.append(f"## {name[:120]}")
        for key, label in METRICS:
            if key in idx:
                lines.append(f"- {label} (`{key}`): {r[idx[key]]} {units[idx[key]]}")
                rec[key] = r[idx[key]] + " " + units[idx[key]]
        out.append(rec)
        lines.append("")
    text = "\n".join(lines)
    if args.out:
        open(args.out, "w").write(text + "\n")
        json.dump(out, open(args.out.rsplit(".", 1)[0] + ".json", "w"), indent=1)
    print(text)


if __name__ == "__main__":
    sys.exit(main())
