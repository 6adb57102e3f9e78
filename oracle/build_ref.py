"""Build the reference's CPU path for the Himeno program into oracle/_ref/.

The reference times a genome by compiling the (annotated) program text with
the user's compile template and running the binary (acctuner/evaluators.py:
190-222).  With gcc the pragmas are ignored, so every genome's binary is the
all-CPU program; this script compiles the same C-subset text
(paper_2002_12115_b200/apps/himeno.py) with the reference template
"gcc -O2 -w" (+ -mcmodel=medium for the >2 GiB static arrays of the large
grids).  Outputs go to oracle/_ref/ only (git-ignored, travels with gpurun).

    python oracle/build_ref.py [SIZE:NN ...]      default: XS:3 M:3 L:1 L:3
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2002_12115_b200.apps import himeno  # noqa: E402

OUT = ROOT / "oracle" / "_ref"


def build(cases=(("XS", 3), ("M", 3), ("L", 1), ("L", 3))):
    OUT.mkdir(parents=True, exist_ok=True)
    built = []
    for name, nn in cases:
        src = OUT / f"himeno_{name.lower()}_n{nn}.c"
        binary = OUT / f"himeno_{name.lower()}_n{nn}"
        text = himeno.source_text(name, nn)
        if not binary.exists() or not src.exists() or src.read_text() != text:
            src.write_text(text)
            subprocess.run(["gcc", "-O2", "-w", "-mcmodel=medium", str(src), "-o", str(binary)],
                           check=True)
        built.append(binary)
    return built


if __name__ == "__main__":
    cases = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]] or None
    for b in (build(cases) if cases else build()):
        print(b)
