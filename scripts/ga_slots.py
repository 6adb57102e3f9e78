"""GA config 4 (M, nn=3, pop 20 x 20, seed 0) with 4 / 8 / 16 concurrent worker slots on
one GPU: generations/s, executed evals/s, per-GPU busy seconds, host CPU load -- the
one-GPU analogue of 8 devices each running an evaluation (host-core contention of the
gene-0 loops)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for host_build in ("tuned", "reference"):
    for w in (4, 8, 16):
        r = bench.ga_throughput(0, "M", 3, 20, 20, 0, w, host_build=host_build)
        keep = {k: r[k] for k in ("workers_per_gpu", "wall_s", "gens_per_s", "executed_evals",
                                  "executed_evals_per_s", "best_genome", "best_time_s",
                                  "per_gpu", "host")}
        keep["host_build"] = host_build
        print(json.dumps(keep), flush=True)
