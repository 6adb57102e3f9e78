"""The C-ABI library loads and exports every symbol include/himeno_b200.h declares.

No compute calls here (no GPU in the dev container); device-less behaviour is
checked: hp_device_count() == 0 and hp_create fails with HP_ERR_DEVICE.
"""
import ctypes as C
import re

import pytest

from conftest import ROOT, has_gpu
from paper_2002_12115_b200 import native as N

HEADER = (ROOT / "include" / "himeno_b200.h").read_text()


def declared():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z_0-9]+)\s*\(", body)))


def test_header_declares_expected_api():
    names = declared()
    for must in ("hp_create", "hp_destroy", "hp_run", "hp_read_field", "hp_last_error",
                 "hp_jacobi_device", "hp_jacobi_host", "hp_time_steps"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) <= set(N.SIGNATURES)


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against the header; every ctypes mirror must match C's layout."""
    import subprocess
    structs = {"hp_grid": N.Grid, "hp_event": N.Event, "hp_schedule": N.Schedule,
               "hp_result": N.Result, "hp_kernel_times": N.KernelTimes}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "himeno_b200.h"',
             "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        cname, field, value = line.split()
        got[(cname, field)] = int(value)
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_abi_version():
    assert N.load().hp_abi_version() == N.ABI_VERSION


@pytest.mark.skipif(has_gpu(), reason="device-less behaviour only")
def test_no_device_behaviour():
    assert N.device_count() == 0
    from paper_2002_12115_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        N.Context(0, 9, 9, 17)


def _build_c_host(tmp_path):
    import subprocess
    exe = tmp_path / "c_host"
    lib_dir = ROOT / "paper_2002_12115_b200" / "_native"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "c_host_example.c"), "-L", str(lib_dir),
                    "-lhimeno_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


@pytest.mark.skipif(has_gpu(), reason="device-less behaviour only")
def test_c_host_links_and_reports_no_device(tmp_path):
    """A plain C program builds against include/himeno_b200.h + the .so (no torch)."""
    import subprocess
    out = subprocess.run([str(_build_c_host(tmp_path))], capture_output=True, text=True)
    assert out.returncode == 2 and "environment" in out.stdout


@pytest.mark.gpu
def test_c_host_runs_on_device(tmp_path):
    import subprocess
    from oracle import oracle
    out = subprocess.run([str(_build_c_host(tmp_path))], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    gosa = float(out.stdout.split()[-1])
    ref = oracle.run_program(33, 33, 65, 3)["gosa64"]
    assert abs(gosa - ref) <= 1e-12 * ref
