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


def test_sample_rows_cover_first_last_and_stride():
    rows = bench.sample_rows(8_000_000, 65536)
    assert rows[0] == 0 and rows[-1] == 8_000_000 - 1
    assert set(range(1024)) <= set(rows[:1100].tolist())
    assert 60000 < rows.size < 70000 and (rows[1:] > rows[:-1]).all()
    assert bench.sample_rows(500, 65536).tolist() == list(range(500))


class _Args:
    def __init__(self, config, shard=None, grid="1x1", scaling=None):
        self.config, self.shard, self.grid, self.scaling = config, shard, grid, scaling


def test_plan_strong_weak_trees_grid():
    c4 = synthetic.CONFIGS[4]
    plans = [bench.Plan(_Args(4), c4, 8, r) for r in range(8)]
    assert all(p.scaling == "strong" and not p.reduce for p in plans)
    assert sum(p.n for p in plans) == c4.n_objects and plans[0].total_objects == c4.n_objects
    assert len({p.data_seed for p in plans}) == 8
    c2 = synthetic.CONFIGS[2]
    p = bench.Plan(_Args(2), c2, 4, 3)
    assert p.scaling == "weak" and p.n == c2.n_objects and p.total_objects == 4 * c2.n_objects
    c5 = synthetic.CONFIGS[5]
    t = [bench.Plan(_Args(5), c5, 4, r) for r in range(4)]
    assert all(q.shard == "trees" and q.reduce and q.n == c5.n_objects for q in t)
    assert [q.tree_range for q in t] == [(0, 1000), (1000, 2000), (2000, 3000), (3000, 4000)]
    assert len({q.data_seed for q in t}) == 1
    g = [bench.Plan(_Args(5, "grid", "2x2"), c5, 4, r) for r in range(4)]
    assert [(q.object_index, q.tree_index) for q in g] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert g[0].n + g[2].n == c5.n_objects and g[0].data_seed == g[1].data_seed != g[2].data_seed
    one = bench.Plan(_Args(5), c5, 1, 0)
    assert one.shard == "objects" and not one.reduce and one.n == c5.n_objects
