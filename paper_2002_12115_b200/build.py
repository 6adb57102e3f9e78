"""Build libhimeno_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2002_12115_b200.build [--force] [--verbose]

* kernels.cu   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
               --fmad=false (bit-exact with the host loops / oracle)
* executor.cpp g++ -O3 -march=x86-64-v3 -ffp-contract=off (AVX2 host loops, no FMA
  contraction: every product and sum rounds separately, as on the device);
  host_loops_ref.cpp g++ -O2 (the reference's compile template, HP_FLAG_HOST_REFERENCE)
* link         nvcc -shared -cudart static  ->  paper_2002_12115_b200/_native/

Generated executors (codegen.py; generic.APPS): for every application text with a
committed program model, ``gen/<app>.cu`` is generated and compiled the same way
into ``_native/libapp_<app>.so``.

The .so files are git-ignored but travel to the GPU box with the gpurun snapshot.
Rebuilds only when a source or header is newer than the library.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_native"
LIB = OUT_DIR / "libhimeno_b200.so"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_home() -> Path:
    for cand in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if cand and (Path(cand) / "bin" / "nvcc").exists():
            return Path(cand)
    nvcc = shutil.which("nvcc")
    if nvcc:
        return Path(nvcc).resolve().parent.parent
    raise RuntimeError("nvcc not found (set CUDA_HOME)")


def _sources() -> list:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    newest = max(p.stat().st_mtime for p in
                 _sources() + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) +
                 sorted(INCLUDE.glob("*.h")) + [Path(__file__)])
    return newest > LIB.stat().st_mtime


def _run(cmd: list, verbose: bool) -> None:
    if verbose:
        print(" ".join(map(str, cmd)), flush=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{proc.stdout}\n{proc.stderr}")
    if verbose and (proc.stdout.strip() or proc.stderr.strip()):
        print(proc.stdout + proc.stderr, flush=True)


GEN_DIR = PKG / "gen"


def _gen_inputs() -> list:
    return [PKG / "codegen.py", CSRC / "gen_runtime.cuh", INCLUDE / "app_b200.h",
            PKG / "apps" / "ft.py", PKG / "apps" / "himeno.py", Path(__file__)] + \
        sorted((PKG / "apps" / "model").glob("*.json"))


def build_apps(force: bool = False, verbose: bool = False) -> list:
    """Generate and compile every generated executor (generic.APPS)."""
    from . import codegen, generic
    cuda = _cuda_home()
    nvcc = str(cuda / "bin" / "nvcc")
    OUT_DIR.mkdir(exist_ok=True)
    GEN_DIR.mkdir(exist_ok=True)
    newest = max(p.stat().st_mtime for p in _gen_inputs())
    specs = generic.app_specs()
    out = []
    for name in generic.APPS:
        lib = generic.lib_path(name)
        out.append(lib)
        if not force and lib.exists() and lib.stat().st_mtime >= newest:
            continue
        spec = specs[name]
        prog = spec.program()
        kinds = {lid: k.value for lid, k in prog.kinds.items()}
        src = GEN_DIR / f"{name}.cu"
        src.write_text(codegen.generate(name, spec.text(), prog.model, kinds))
        tmp = lib.with_suffix(".so.tmp")
        _run([nvcc, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-diag-suppress", "177,550,549",
              "-I", str(INCLUDE), "-I", str(CSRC), "-shared", "-cudart", "static",
              "-o", str(tmp), str(src)], verbose)
        os.replace(tmp, lib)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    build_apps(force, verbose)
    if not force and not _stale():
        return LIB
    cuda = _cuda_home()
    nvcc = str(cuda / "bin" / "nvcc")
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    inc = ["-I", str(INCLUDE), "-I", str(CSRC)]
    for src in sorted(CSRC.glob("*.cu")):
        obj = OUT_DIR / (src.stem + ".o")
        extra = os.environ.get("HP_EXTRA_NVCC_FLAGS", "").split()   # experiment builds only
        _run([nvcc, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3", *extra,
              *inc, "-c", str(src), "-o", str(obj)], verbose)
        objs.append(obj)
    for src in sorted(CSRC.glob("*.cpp")):
        obj = OUT_DIR / (src.stem + ".o")
        # *_ref.cpp: the reference's compile template (`gcc -O2 -w`, evaluators.py:154-165):
        # the reference-faithful host build of the loops (HP_FLAG_HOST_REFERENCE)
        opt = ["-O2"] if src.stem.endswith("_ref") else ["-O3", "-march=x86-64-v3"]
        _run(["g++", *opt, "-std=c++17", "-fPIC", "-ffp-contract=off",
              "-fno-fast-math",
              "-Wall", "-Wno-unused-function", "-I", str(cuda / "include"), *inc,
              "-c", str(src), "-o", str(obj)], verbose)
        objs.append(obj)
    tmp = LIB.with_suffix(".so.tmp")
    _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs),
          "-Xlinker", "-soname=libhimeno_b200.so", "-ldl"], verbose)
    os.replace(tmp, LIB)
    for obj in objs:
        obj.unlink(missing_ok=True)
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args(argv)
    lib = build(force=args.force, verbose=args.verbose)
    print(lib)
    return 0


if __name__ == "__main__":
    sys.exit(main())
