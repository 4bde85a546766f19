"""The bench's roofline models (CPU only): the expected wavefronts of a warp-wide random
gather and the B200 shared-memory + HBM floor of a predict."""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2211_00391_b200 import synthetic  # noqa: E402


def test_gather_wavefronts():
    assert bench.gather_wavefronts(128) == 1.0           # 32 words: one per bank
    assert bench.gather_wavefronts(256) == pytest.approx(2.0, abs=0.01)  # 64 fp32 leaves: nearly always 2
    w1k = bench.gather_wavefronts(1024)                   # 256 fp32 leaves
    assert 2.9 < w1k < 3.5


def test_roofline_smem_cfg2():
    spec = synthetic.WorkloadSpec("cfg2", 1_000_000, 200, 64, 2000, 6, 0.05, cfg=2)
    r = bench.roofline_smem(spec, 148, 1965e6, 6545.9, 4)
    # 6/128 + 2/32 wavefronts per object-tree at one per SM per clock
    assert r["wavefronts_per_object_tree"] == pytest.approx(6 / 128 + 2 / 32, rel=0.01)
    assert r["t_apply_floor_ms"] == pytest.approx(2e9 * r["wavefronts_per_object_tree"] / (148 * 1965e6) * 1e3)
    assert r["t_quantize_floor_ms"] == pytest.approx(1e9 / 6545.9e9 * 1e3)
