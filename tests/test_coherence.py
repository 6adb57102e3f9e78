"""Data-manager coherence algebra (csrc/coherence.h), compiled with g++ and run on CPU."""
import subprocess

from conftest import ROOT


def test_coherence_driver(tmp_path):
    exe = tmp_path / "coh"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", "/usr/local/cuda/include",
                    "-I", str(ROOT / "include"), "-I", str(ROOT / "paper_2002_12115_b200" / "csrc"),
                    str(ROOT / "tests" / "coherence_driver.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "OK", out.stdout + out.stderr
