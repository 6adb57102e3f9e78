"""bench.py helpers that run without a GPU: the roofline denominator lookup."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def test_peaks_fallback_without_measured_file(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    peak, src = bench.peaks()
    assert peak == 6650.0 and src.startswith("fallback")


def test_peaks_prefers_sustained_hbm_figure(tmp_path, monkeypatch):
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps(
        {"hbm_gbs": {"burst": 7100.0, "sustained": 6548.0}, "bf16_tflops": 1800.0}))
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    peak, src = bench.peaks()
    assert peak == 6548.0 and "sustained" in src


def test_peaks_flat_key_and_tbs_units(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_gbs": 6600.0}))
    assert bench.peaks()[0] == 6600.0
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_copy_tbs": 6.5}))
    assert bench.peaks()[0] == 6500.0


def test_peaks_ignores_flops_entries(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"bf16_tflops": 1800.0}))
    assert bench.peaks()[1].startswith("fallback")
