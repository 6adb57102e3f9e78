"""The all-CPU program and the GA on M under both host builds of the gene-0 loops
(tuned vs the reference's compile template): program times and where the GA lands."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2002_12115_b200.evaluator import B200Evaluator  # noqa: E402

for build in ("tuned", "reference"):
    with B200Evaluator("M", nn=3, host_build=build) as ev:
        t = {g: min(ev.measure(tuple(int(c) for c in g)).seconds for _ in range(3))
             for g in ("0" * 13, "0000000100100", "1001000000000", "1001001000000")}
    print(json.dumps({"host_build": build, "program_s": t}), flush=True)
