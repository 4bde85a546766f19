"""The N>1 path with the GPU evaluator on a 1-GPU box: ranks share cuda:0 and talk over
gloo (a functional check of the multi-rank code -- never a measurement; the sharded
classes and bench.py use NCCL on a multi-GPU node).  Each rank runs the sm_100a
kernels; results are checked against the CPU oracle."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2211_00391_b200 as obt
from paper_2211_00391_b200 import multiclass, sharding, synthetic

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _multi_model():
    spec = synthetic.WorkloadSpec("m", 1, 24, 60, 203, 9, 0.01, n_outputs=10, cfg=5)
    return multiclass.from_arrays(synthetic.model_arrays(spec, seed=11, affine=True))


def _flat_multi(mm):
    counts = np.array([b.size for b in mm.borders], np.int32)
    borders = np.full((mm.n_features, int(counts.max())), np.inf, np.float32)
    for f, b in enumerate(mm.borders):
        borders[f, : b.size] = b
    return oracle.FlatModel(borders, counts, np.full(mm.n_trees, mm.depth, np.int32), mm.split_feature,
                            mm.split_ordinal, mm.leaves, mm.scale, mm.bias)


def _worker(rank, world, port, case):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = synthetic.WorkloadSpec("t", 1, 24, 60, 301, 7, 0.1, cfg=1)
        model = synthetic.build_model(spec, seed=5, affine=True)
        x = synthetic.host_features(synthetic.WorkloadSpec("t", 5000, 24, 1, 1, 1, 0.1, cfg=1), seed=6)
        x = synthetic.sprinkle_specials(x, [ff.borders for ff in model.float_features], seed=7)
        m = obt.FeatureMatrix(x, obt.Layout.OBJECT_MAJOR)
        if case == "objects":
            full = oracle.evaluate_scalar(oracle.flatten(model), x)
            ev = sharding.ObjectShardedEvaluator(model, device=0)
            assert np.array_equal(ev.predict(m), full), "GPU object sharding must be bit-exact"
            b, e = sharding.object_shard(x.shape[0], rank, world)
            local = ev.predict_device(torch.from_numpy(x[b:e]).cuda())
            assert np.array_equal(local.cpu().numpy(), full[b:e])
        elif case == "trees":
            full = oracle.evaluate_scalar(oracle.flatten(model), x)
            ev = sharding.TreeShardedEvaluator(model, device=0)
            for got in (ev.predict(m), ev.predict_device(torch.from_numpy(x).cuda()).cpu().numpy()):
                rel = np.abs(got - full) / np.maximum(np.maximum(np.abs(got), np.abs(full)), 1e-300)
                assert rel.max() <= 1e-12, rel.max()
        else:
            mm = _multi_model()
            full = oracle.evaluate_scalar(_flat_multi(mm), x)
            go, gt = (1, 2) if case == "grid_trees" else (2, 1)
            ev = sharding.GridShardedEvaluator(mm, go, gt, device=0)
            got = ev.predict(m)
            assert got.shape == full.shape == (x.shape[0], 10)
            rel = np.abs(got - full) / np.maximum(np.maximum(np.abs(got), np.abs(full)), 1e-300)
            assert rel.max() <= 1e-12, rel.max()
            if gt == 1:
                assert np.array_equal(got, full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["objects", "trees", "grid_trees", "grid_objects"])
def test_two_ranks_gpu_evaluator(case):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), case), nprocs=2, join=True)


@pytest.mark.parametrize("config,extra", [(1, []), (5, ["--objects", "20000", "--trees", "64"]),
                                          (5, ["--objects", "20000", "--trees", "64", "--leaves", "fp16"])])
def test_bench_self_spawns_two_ranks(config, extra):
    """`bench.py --gpus 2` launches two ranks itself (gloo on one GPU here); the line
    reports n_gpus 2 and a verified timed batch."""
    env = {**os.environ, "OBT_BENCH_DIST_BACKEND": "gloo"}
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", str(config), "--steps", "3",
           "--warmup", "3", "--no-e2e", *extra]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    assert line["verify"]["passed"] and line["verify"]["ranks"] == 2
    if config == 5:
        assert line["config"]["shard"] == "trees" and line["nccl_reduce_ms"] is not None


def test_both_bench_arms_print_the_same_config():
    """The reference arm (`--impl reference`) names the same workload and partitioning as
    our arm, key for key, so the driver's ratio compares like with like."""
    def line(extra):
        cmd = [sys.executable, str(ROOT / "bench.py"), "--config", "1", "--steps", "3", "--warmup", "3", *extra]
        res = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
        assert res.returncode == 0, res.stderr[-4000:]
        return json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])

    ours = line(["--no-e2e", "--no-cpu-baseline"])
    ref = line(["--impl", "reference", "--no-reference-pkg"])
    assert ref["impl"] == "reference" and "impl" not in ours
    assert ours["config"] == ref["config"]
    for key in ("metric", "unit", "higher_is_better", "scaling", "n_gpus", "steps", "warmup"):
        assert ours[key] == ref[key], key
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["cpu_baseline"]["kind"] == "port"
