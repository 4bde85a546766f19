#!/usr/bin/env python
"""Benchmark: object-trees/s of oblivious-ensemble predict on B200, with roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One "step" is one predict over one batch of the workload.  The default workload is
BASELINE.json configs[3] (config 4: 8,000,000 objects x 500 features, 128 borders,
8,000 depth-8 trees, fp32 leaves) -- the largest configuration that runs on one GPU,
"objects sharded over 1/2/4/8 GPUs": at N GPUs each rank owns 8M/N of the objects
(strong scaling, no data-path collective).  Configs 1-3 default to weak scaling (every
rank its own batch of the configuration's size); config 5 shards trees (NCCL
all_reduce of binary64 partials + finalize inside every step), or objects / a 2-D grid
with --shard.  `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).

Printed on rank 0 as ONE JSON line:
  value      whole-job object-trees/s, features resident in HBM, CUDA-event timed
  verify     the timed batch's outputs (a strided sample of ~64k rows from every rank,
             first and last tiles included) against the CPU oracle: bit-exact flag
  e2e        the same metric through Evaluator.predict with pinned host buffers
             (host->device features and device->host scores inside the timed region);
             e2e_pageable: the literal drop-in call (numpy input, fresh output)
  roofline   the dominant kernel (tree apply) against the integer-issue peak, plus the
             whole-step roofline of SURVEY.md section 8d
  cpu_baseline  the C oracle port of the reference algorithm on this host's cores, and
             (reference_pkg) the reference package itself, 1 core and all cores
  fp16_vs_fp32  (config 3) deviation metrics / flips of the fp16-leaf predictions
`--impl reference` times the CPU port alone on the same config and metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "object-trees/sec for oblivious-ensemble predict at 1/2/4/8 B200; % roofline"
UNIT = "object-trees/s"
FALLBACK_HBM_GBS = 6650.0
FALLBACK_SM_MHZ = 1965.0


def quantize_search(ev, n_features: int) -> str:
    """The predict path's quantize search: cells(k) = cell-table kernel with k compares
    per value, eytzinger(L) = L-level search; rows that are not 16-byte multiples
    (F % 4 != 0) take the LDG-loaded Eytzinger kernel instead of the TMA-staged ones."""
    if n_features % 4:
        return "eytzinger (LDG rows: F % 4 != 0)"
    if not hasattr(ev, "quantize_kernel"):
        return "n/a"
    kind, param = ev.quantize_kernel()
    return f"{kind}({param})"


def peaks() -> dict:
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        data = json.loads(path.read_text())
        return {"hbm_gbs": float(data["hbm_gbs"]), "sm_max_mhz": float(data.get("sm_max_mhz", FALLBACK_SM_MHZ)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": FALLBACK_SM_MHZ, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._reader = threading.Thread(target=self._read, daemon=True)
            self._reader.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self, t0: float, t1: float) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            rows.append((ts, parts))
        inside = [r for r in rows if t0 <= r[0] <= t1 + 0.06] or rows[-3:]
        sm = sorted(float(p[0]) for _, p in inside if p[0].replace(".", "").isdigit())
        smax = [float(p[1]) for _, p in inside if p[1].replace(".", "").isdigit()]
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        reasons = sorted({names[i] for _, p in inside for i in range(4) if p[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(inside)}


# NCCL on GPUs.  OBT_BENCH_DIST_BACKEND=gloo is a functional check of the multi-rank code
# path on a box with fewer GPUs than ranks (ranks then share devices: never a measurement).
DIST_BACKEND = os.environ.get("OBT_BENCH_DIST_BACKEND", "nccl")


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if DIST_BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(DIST_BACKEND)
    return world, rank, local


def reduce_device() -> str:
    return "cuda" if DIST_BACKEND == "nccl" else "cpu"


def max_over_ranks(value: float, world: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def roofline_terms(spec) -> dict:
    """bytes = 4NF + 8NC, ops = NTD + NF*ceil(log2(B+1)) + NTC."""
    N, F, B, T, D, C = spec.n_objects, spec.n_features, spec.borders, spec.n_trees, spec.depth, spec.n_outputs
    return {
        "bytes": 4 * N * F + 8 * N * C,
        "ops": N * T * D + N * F * math.ceil(math.log2(B + 1)) + N * T * C,
        "apply_ops": N * T * D + N * T * C,
        "quantize_bytes": 4 * N * F + N * F,
    }


def gather_wavefronts(table_bytes: int, trials: int = 4000, seed: int = 7) -> float:
    """Expected shared-memory wavefronts of one warp-wide random gather from a table of
    `table_bytes` (4-byte banks, 32 banks, 32 lanes, uniform random 4-byte words; a
    wavefront serves one distinct word per bank): E[max over banks of distinct words]."""
    import numpy as np

    words = max(1, table_bytes // 4)
    if words <= 32:
        return 1.0
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, words, size=(trials, 32))
    total = 0
    for row in idx:
        u = np.unique(row)
        total += np.bincount(u % 32, minlength=32).max()
    return total / trials


def roofline_smem(spec, n_sm: int, sm_hz: float, hbm_gbs: float, leaf_bytes: int) -> dict:
    """The B200 floor of this path: the apply kernel is bound by the
    shared-memory pipe -- one 128-byte wavefront per SM per clock -- at D bucket bytes per
    object-tree (a warp's 32 lanes x 4 objects read 128 bytes per depth) plus one random
    gather per object-tree from a 2^D-leaf table; the quantize by HBM (4NF read + NF
    written).  Single-output configs; the two phases are serial within a predict."""
    N, F, T, D = spec.n_objects, spec.n_features, spec.n_trees, spec.depth
    wf_per_ot = D / 128.0 + gather_wavefronts((1 << D) * leaf_bytes) / 32.0
    t_apply = N * T * wf_per_ot / (n_sm * sm_hz)
    t_quant = (4 * N * F + N * F) / (hbm_gbs * 1e9)
    return {"t_apply_floor_ms": t_apply * 1e3, "t_quantize_floor_ms": t_quant * 1e3,
            "wavefronts_per_object_tree": wf_per_ot,
            "model": "apply: shared-memory wavefronts (1 per SM per clock); quantize: HBM bytes"}


def reduce_over_ranks(values, world: int, op: str):
    """Element-wise MAX / MIN / SUM of a list of floats over ranks."""
    if world == 1:
        return list(values)
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=reduce_device())
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op])
    return [float(v) for v in t.cpu()]


def free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(argv, n: int) -> int:
    """`--gpus N` outside torchrun: re-launch this script as N ranks on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def flat_model(model):
    """The oracle's flat layout for an ObliviousModel or a multiclass.MultiOutputModel."""
    import numpy as np

    import oracle

    if not hasattr(model, "subset"):
        return oracle.flatten(model)
    counts = np.array([b.size for b in model.borders], np.int32)
    borders = np.full((model.n_features, max(1, int(counts.max()))), np.inf, np.float32)
    for f, b in enumerate(model.borders):
        borders[f, : b.size] = b
    return oracle.FlatModel(borders, counts, np.full(model.n_trees, model.depth, np.int32), model.split_feature,
                            model.split_ordinal, model.leaves, model.scale, model.bias)


def sample_rows(n: int, target: int, edge: int = 1024):
    """Deterministic rows of an n-object batch: the first and last `edge` rows (first and
    last tiles) and every k-th row, about `target` in all, sorted and unique."""
    import numpy as np

    if n <= target:
        return np.arange(n, dtype=np.int64)
    step = max(1, n // max(1, target - 2 * edge))
    rows = np.concatenate([np.arange(min(edge, n)), np.arange(max(0, n - edge), n), np.arange(0, n, step)])
    return np.unique(rows.astype(np.int64))


def verify_timed(x, out, fm, precision: int, rows, exact: bool) -> dict:
    """The timed batch's outputs on `rows` against the CPU oracle on the same feature rows."""
    import numpy as np
    import torch

    import oracle

    idx = torch.from_numpy(rows).to(x.device)
    xs = x.index_select(0, idx).cpu().numpy()
    got = out.index_select(0, idx).cpu().numpy()
    oracle.set_threads(oracle.host_cores())
    want = oracle.evaluate_scalar(fm, xs, oracle.OBJECT_MAJOR, precision)
    want = want.reshape(got.shape)
    rel = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1e-300)
    rel = np.where(got == want, 0.0, rel)
    ab = np.where(got == want, 0.0, np.abs(got - want))
    return {"rows": int(rows.size), "bit_exact": bool(np.array_equal(got, want)),
            "max_rel_dev": float(np.nanmax(rel)) if rel.size else 0.0,
            "max_abs_dev": float(np.nanmax(ab)) if ab.size else 0.0, "expect_bit_exact": exact}


def cpu_baseline_port(spec, fm, x, trees: int, seconds: float) -> dict:
    """The C oracle port of the reference algorithm on all host cores, on a prefix of the
    timed batch's rows (doubling until one pass takes >= seconds/4)."""
    import oracle

    oracle.set_threads(oracle.host_cores())  # all host cores, whatever OMP_NUM_THREADS says
    prec = oracle.BINARY16 if spec.half_leaves else oracle.BINARY64
    n_max = x.shape[0]
    n = min(4096, n_max)
    while True:
        xs = x[:n].cpu().numpy()
        t0 = time.perf_counter()
        oracle.evaluate_scalar(fm, xs, oracle.OBJECT_MAJOR, prec)
        dt = time.perf_counter() - t0
        if dt >= seconds / 4 or n >= n_max or n >= 1 << 22:
            break
        n = min(n_max, 2 * n)
    reps = max(1, int(round(seconds * 0.75 / max(dt, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.evaluate_scalar(fm, xs, oracle.OBJECT_MAJOR, prec)
    dt = (time.perf_counter() - t0) / reps
    return {
        "value": n * trees / dt, "unit": UNIT, "cores": oracle.max_threads(), "host_cpus": os.cpu_count(),
        "kind": "port",
        "sample": f"the first {n} of the timed batch's {n_max} objects (full {trees}-tree model), {reps} reps; "
                  f"C restatement of evaluate_scalar (oracle/obtree_oracle.c), OpenMP over objects",
    }


REF_PKG = ROOT / "baseline" / "_ref"


def reference_model(model):
    """The reference package's ObliviousModel for one of ours (same values)."""
    import numpy as np

    import obtree

    ff = tuple(obtree.FloatFeatureBorders(f.feature_index, np.asarray(f.borders, np.float32))
               for f in model.float_features)
    trees = tuple(obtree.ObliviousTree(t.depth, tuple(obtree.SplitCondition(s.feature_index, s.border_ordinal)
                                                      for s in t.splits), np.asarray(t.leaf_values))
                  for t in model.trees)
    return obtree.ObliviousModel(ff, trees, model.scale, model.bias)


def refpkg_worker(path: str, core: int, offset: int, n: int, half: bool) -> None:
    """One pinned process timing the reference package's Evaluator (its own _time_case)."""
    import numpy as np

    os.sched_setaffinity(0, {core})
    sys.path.insert(0, str(REF_PKG))
    import obtree
    from obtree.bench import _time_case

    from paper_2211_00391_b200 import synthetic

    data = np.load(path, allow_pickle=False)
    spec = synthetic.WorkloadSpec(**json.loads(str(data["spec"])))
    model = reference_model(synthetic.build_model(spec))
    x = np.ascontiguousarray(data["x"][offset: offset + n])
    cfg = (obtree.EvalConfig(block_size=512, strategy=obtree.LeafStrategy.NAIVE16) if half else obtree.EvalConfig())
    ev = obtree.Evaluator(model, cfg)
    fm = obtree.FeatureMatrix(x, obtree.Layout.OBJECT_MAJOR)
    ev.predict(fm)  # warm-up (the reference bench's verification run)
    mean, std, inner = _time_case(ev, fm, 3)
    print(json.dumps({"seconds": mean, "std": std, "inner": inner, "n": int(x.shape[0]), "core": core}), flush=True)


def reference_pkg_baseline(spec, x, budget_s: float) -> dict:
    """The reference package itself (pure Python + numpy, installed into baseline/_ref by
    pip from /root/reference/pkg) on this host: 1 core, then one pinned process per core
    each on its own slice of the timed batch (the reference is single-threaded by
    contract), timed by the reference's own bench._time_case
    (process_time, doubling inner loop, 3 repetitions)."""
    import tempfile

    import numpy as np

    if not (REF_PKG / "obtree").exists():
        return {"unavailable": "baseline/_ref/obtree not installed (pip install --target baseline/_ref)"}
    if spec.n_outputs > 1 or spec.depth > 8:
        return {"unavailable": "the reference stops at depth 8 and one output (model.py:22, SPEC.md:15)"}
    cores = sorted(os.sched_getaffinity(0))
    # ~35 us per object per 1000 depth-8 trees on one core (measured here): ~0.6 s slices
    per_obj = 3.5e-5 * spec.n_trees / 1000.0
    n = int(max(64, min(4096, 0.6 / per_obj)))
    n_all = min(x.shape[0], n * len(cores))
    xs = x[:n_all].cpu().numpy()
    fd, path = tempfile.mkstemp(suffix=".npz")
    os.close(fd)
    fields = {k: getattr(spec, k) for k in spec.__dataclass_fields__}
    np.savez(path, x=xs, spec=np.array(json.dumps(fields)))
    env = {**os.environ, "OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"}

    def launch(core, offset):
        return subprocess.Popen([sys.executable, str(Path(__file__).resolve()), "--refpkg-worker", path, str(core),
                                 str(offset), str(n), "1" if spec.half_leaves else "0"],
                                stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env)

    def collect(procs):
        res = []
        for p in procs:
            try:
                o, e = p.communicate(timeout=budget_s)
            except subprocess.TimeoutExpired:
                p.kill()
                continue
            if p.returncode == 0 and o.strip():
                res.append(json.loads(o.strip().splitlines()[-1]))
        return res

    try:
        one = collect([launch(cores[0], 0)])
        if not one:
            return {"unavailable": "reference worker failed"}
        slots = [c for c in cores if (cores.index(c) + 1) * n <= n_all]
        allr = collect([launch(c, i * n) for i, c in enumerate(slots)])
    finally:
        os.unlink(path)
    v1 = one[0]["n"] * spec.n_trees / one[0]["seconds"]
    vall = sum(r["n"] * spec.n_trees / r["seconds"] for r in allr)
    cfg = "EvalConfig(block_size=512, strategy=NAIVE16)" if spec.half_leaves else "EvalConfig() (block 128, W512, NAIVE)"
    return {"value_1core": v1, "value_all_cores": vall, "unit": UNIT, "cores": len(allr), "kind": "reference",
            "impl": "obtree 0.1.0 Evaluator.predict (the reference package, pure Python + numpy) with " + cfg,
            "timer": "obtree.bench._time_case (process CPU time, per pinned process)",
            "sample": f"{n} objects of the timed batch per process (disjoint slices), full {spec.n_trees}-tree model"}


def fp16_report(model, x, p16, device: int) -> dict:
    """Config 3 (and --leaves fp16): the fp16-leaf predictions of the timed batch against
    the fp32-leaf ones (reference oracle.py:57-92 metrics, flips at threshold 0, and the
    reference's bound |scale| * T * max|leaf| * 2^-10 of test_acceptance.py:156); for a
    multi-output model over every (object, output)."""
    import numpy as np

    import paper_2211_00391_b200 as obt

    if hasattr(model, "subset"):
        from paper_2211_00391_b200 import multiclass

        ev32 = multiclass.MultiOutputEvaluator(model, device=device)
        from paper_2211_00391_b200.model import half_bank_values

        halves, sat = half_bank_values(model.leaves)
        max_abs, sat_count = float(np.max(np.abs(halves.astype(np.float64)))), sat
    else:
        ev32 = obt.Evaluator(model, obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE), device=device)
        bank = obt.build_leaf_bank(model, obt.LeafPrecision.BINARY16)
        max_abs, sat_count = bank.max_abs_leaf, bank.saturation_count
    p32 = ev32.predict_device(x).cpu().numpy().ravel()
    p16 = p16.cpu().numpy().ravel()
    m = obt.deviation_metrics(p32, p16)
    bound = abs(model.scale) * model.n_trees * max_abs * 2.0 ** -10
    return {"vs": "fp32-leaf (binary64-fold) predictions of the same timed batch", "objects": int(p16.size),
            "max_abs": m.max_abs, "mean_abs": m.mean_abs, "median_abs": m.median_abs, "rms": m.rms,
            "flips_at_0": obt.classification_flip_count(p32, p16, 0.0), "bound": bound,
            "within_bound": bool(m.max_abs <= bound), "saturated_leaves": sat_count}


def workload_config(spec, plan, world) -> dict:
    """`config` of the JSON line: the workload and how it is partitioned -- the same dict
    on both arms (ours and --impl reference), so the driver compares like with like.
    What is specific to the GPU path (kernels chosen, per-GPU shares) goes in `device_path`."""
    go, gt = plan.grid
    per_gpu = plan.n
    return {"workload": spec.name, "n_objects_total": plan.total_objects, "features": spec.n_features,
            "borders": spec.borders, "trees": spec.n_trees, "depth": spec.depth, "outputs": spec.n_outputs,
            "leaves": "fp16 (binary32 fold)" if spec.half_leaves else "fp32 values (binary64 fold)",
            "l2": ("inputs larger than L2 (features 4NF bytes, buckets NF bytes > 126 MB)"
                   if 4 * per_gpu * spec.n_features > 126e6 else
                   "inputs L2-resident between steps (features 4NF bytes < 126 MB; a launch-bound size)"),
            "parallelism": plan.parallelism(world), "shard": plan.shard}


def run_reference(args, world, rank):
    """--impl reference: the CPU port of the reference algorithm, all host threads."""
    if rank != 0:
        return
    import oracle
    from paper_2211_00391_b200 import synthetic

    spec = synthetic.CONFIGS[args.config]
    if args.leaves:
        spec = synthetic.WorkloadSpec(**{**spec.__dict__, "half_leaves": args.leaves == "fp16",
                                         "name": spec.name + ("-fp16" if args.leaves == "fp16" else "")})
    if spec.n_outputs > 1:
        from paper_2211_00391_b200 import multiclass

        model = multiclass.from_arrays(synthetic.model_arrays(spec))
    else:
        model = synthetic.build_model(spec)
    fm = flat_model(model)
    plan = Plan(args, spec, world, rank)
    oracle.set_threads(oracle.host_cores())  # torchrun exports OMP_NUM_THREADS=1; use every core
    prec = oracle.BINARY16 if spec.half_leaves else oracle.BINARY64
    n = min(args.ref_sample, spec.n_objects)
    x = synthetic.host_features(spec, n_objects=n, seed=spec.data_seed + 7)
    for _ in range(args.warmup):
        oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, prec)
        times.append(time.perf_counter() - t0)
    step = sum(times) / len(times)
    value = n * spec.n_trees / step
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": plan.scaling,
        "vs_baseline": None, "dtype": "f16/f32" if spec.half_leaves else "f64",
        "data": "synthetic (seeded; BASELINE names no dataset)",
        "config": workload_config(spec, plan, world),
        "sample_objects_per_step": n,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.max_threads(), "host_cpus": os.cpu_count(),
                         "kind": "port",
                         "sample": f"{n} objects per step drawn with the workload's generator ({spec.name}); the C "
                                   f"restatement of the reference algorithm (oracle/obtree_oracle.c), OpenMP over "
                                   f"objects -- faster per core than the reference package (bench.py's "
                                   f"cpu_baseline.reference_pkg times that one too)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_reference_pkg:
        # the reference package itself (pure Python + numpy from baseline/_ref), 1 core and
        # one pinned process per core, beside the C port this line's value times
        import torch

        line["cpu_baseline"]["reference_pkg"] = reference_pkg_baseline(spec, torch.from_numpy(x), args.cpu_seconds * 4)
    print(json.dumps(line), flush=True)


class Plan:
    """What this rank evaluates: objects (n, data seed) and trees (model), and how the
    step completes (a reduce group for tree / grid sharding)."""

    def __init__(self, args, spec, world, rank):
        from paper_2211_00391_b200 import sharding

        self.multi = spec.n_outputs > 1
        self.shard = args.shard or ("trees" if self.multi and world > 1 else "objects")
        if self.shard == "objects" and not self.multi and args.config in (1, 2, 3) and args.scaling != "strong":
            self.scaling = "weak"
        elif self.shard == "objects" and args.scaling == "weak":
            self.scaling = "weak"
        else:
            self.scaling = "strong"
        go, gt = 1, 1
        if self.shard == "objects":
            go = world
        elif self.shard == "trees":
            gt = world
        else:
            go, gt = (int(v) for v in args.grid.split("x"))
            if go * gt != world:
                raise SystemExit(f"--grid {args.grid} needs {go * gt} ranks, got {world}")
        self.grid = (go, gt)
        self.object_index, self.tree_index = divmod(rank, gt)
        if self.scaling == "weak":
            self.n = spec.n_objects
            self.total_objects = spec.n_objects * go
        else:
            b, e = sharding.balanced_ranges(spec.n_objects, go, quantum=256)[self.object_index]
            self.n = e - b
            self.total_objects = spec.n_objects
        self.tree_range = sharding.tree_shard(spec.n_trees, self.tree_index, gt)
        # ranks of one object shard see the same rows; different shards different rows
        self.data_seed = spec.data_seed + 1000 * self.object_index
        self.reduce = gt > 1

    def parallelism(self, world) -> str:
        go, gt = self.grid
        if self.shard == "objects":
            how = "objects sharded" if self.scaling == "strong" else "one batch per GPU (weak)"
            return f"{how} over {world} GPU(s), no data-path collective"
        if self.shard == "trees":
            return (f"trees sharded over {world} GPU(s); NCCL all_reduce of fp64 partials + finalize inside every "
                    "timed step")
        return (f"{go} object shards x {gt} tree shards; all_reduce of fp64 partials within each object shard + "
                "finalize inside every timed step")


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import oracle
    import paper_2211_00391_b200 as obt
    from paper_2211_00391_b200 import _native, sharding, synthetic

    spec = synthetic.CONFIGS[args.config]
    for kv in args.path:
        name, value = kv.split("=", 1)
        _native.set_path_option(name, int(value))
    if args.objects:
        spec = synthetic.WorkloadSpec(**{**spec.__dict__, "n_objects": args.objects})
    if args.trees:
        spec = synthetic.WorkloadSpec(**{**spec.__dict__, "n_trees": args.trees})
    if args.leaves:
        spec = synthetic.WorkloadSpec(**{**spec.__dict__, "half_leaves": args.leaves == "fp16",
                                         "name": spec.name + ("-fp16" if args.leaves == "fp16" else "")})
    device = local
    torch.cuda.set_device(device)
    plan = Plan(args, spec, world, rank)
    multi = plan.multi
    tb, te = plan.tree_range
    if multi:
        from paper_2211_00391_b200 import multiclass

        full_model = multiclass.from_arrays(synthetic.model_arrays(spec))
        config = obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16) if spec.half_leaves else None
    else:
        full_model = synthetic.build_model(spec)
        config = obt.EvalConfig(strategy=obt.LeafStrategy.NAIVE16 if spec.half_leaves else obt.LeafStrategy.NAIVE)
    sharded, group = None, None
    if plan.reduce:
        # tree / grid sharding through the public sharded evaluator (its inner GPU
        # evaluator holds this rank's tree shard with scale 1 / bias 0)
        sharded = sharding.GridShardedEvaluator(full_model, *plan.grid, config=config, device=device)
        ev, group = sharded.trees.local_evaluator, sharded.trees.group
    elif multi:
        ev = multiclass.MultiOutputEvaluator(full_model, device=device, config=config)
    else:
        ev = obt.Evaluator(full_model, config, device=device)
    x = synthetic.device_features(spec, n_objects=plan.n, seed=plan.data_seed, device=f"cuda:{device}")
    N = plan.n
    out = torch.empty((N, spec.n_outputs) if multi else N, dtype=torch.float64, device=x.device)
    ws = torch.empty(ev.workspace_bytes(N), dtype=torch.uint8, device=x.device)

    def complete():
        # tree / grid sharding: a prediction is complete only after the sum of the ranks'
        # binary64 partials and the affine finalize, so both are part of every step
        if plan.reduce:
            sharding._all_reduce_sum(out, group)
            sharding._finalize_(out, full_model.scale, full_model.bias)

    for _ in range(args.warmup):
        ev.predict_device(x, out=out, workspace=ws)
        complete()
    torch.cuda.synchronize()

    stream = _native.current_stream_handle(device)
    K = args.steps
    t_start, t_end = _native.Event(), _native.Event()
    # launch-bound steps (cfg1: ~30 us of kernels) replay a CUDA graph of one predict, so
    # the number is the GPU's, not the host's launch rate
    t_start.record(stream)
    ev.predict_device(x, out=out, workspace=ws)
    t_end.record(stream)
    torch.cuda.synchronize()
    one_ms = t_start.elapsed_ms(t_end)
    use_graph = not plan.reduce and (args.graph == "on" or (args.graph == "auto" and one_ms < 0.2))
    graph, graph_launches = None, 0
    if use_graph:
        gs = torch.cuda.Stream(device)
        gs.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(gs):
            ev.predict_device(x, out=out, workspace=ws)
        gs.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            ev.predict_device(x, out=out, workspace=ws)
        graph_launches = ev.last_launch_count()
        graph.replay()
        torch.cuda.synchronize()
    marks = [[_native.Event(), _native.Event(), _native.Event()] for _ in range(K if graph is None else min(K, 20))]
    clocks = ClockSampler(device)
    clocks.start()
    time.sleep(0.15)
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t_start.record(stream)
    launches = 0
    for k in range(K):
        if graph is not None:
            graph.replay()
            launches += graph_launches
            continue
        ev.predict_device_marked(x, marks[k], out=out, workspace=ws)
        launches += ev.last_launch_count()
        complete()
    t_end.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier(world)
    clk = clocks.stop(w0, w1)
    elapsed_ms = max_over_ranks(t_start.elapsed_ms(t_end), world)
    step_s = elapsed_ms / K / 1e3
    value = plan.total_objects * spec.n_trees / step_s

    # --- the timed batch's outputs against the oracle (out holds the last timed step)
    fm_full = flat_model(full_model)
    prec = oracle.BINARY16 if spec.half_leaves else oracle.BINARY64
    rows = sample_rows(N, max(1024, args.verify_rows // (8 if multi else 1)))
    ver = verify_timed(x, out, fm_full, prec, rows, exact=not plan.reduce)
    red = reduce_over_ranks([ver["rows"]], world, "sum")
    mx = reduce_over_ranks([ver["max_rel_dev"]], world, "max")[0]
    mabs = reduce_over_ranks([ver["max_abs_dev"]], world, "max")[0]
    mn = reduce_over_ranks([1.0 if ver["bit_exact"] else 0.0], world, "min")[0]
    # tree / grid sharding reassociates the fold: binary64 partials within 1e-12 relative;
    # binary32 partials (binary16 family) within the reference's FP16 acceptance bound
    # |scale| * T * max|leaf| * 2^-10 (test_acceptance.py:156), absolute
    if plan.reduce and spec.half_leaves:
        from paper_2211_00391_b200.model import half_bank_values

        halves = half_bank_values(full_model.leaves if multi else np.concatenate(
            [np.asarray(t.leaf_values, np.float64) for t in full_model.trees]) if full_model.n_trees else np.zeros(1))[0]
        bound = abs(full_model.scale) * spec.n_trees * float(np.max(np.abs(halves.astype(np.float64)))) * 2.0 ** -10
        tol, passed = {"abs": bound}, bool(mabs <= bound)
    elif plan.reduce:
        tol, passed = {"rel": 1e-12}, bool(mx <= 1e-12)
    else:
        tol, passed = 0.0, bool(mn == 1.0)
    verify = {"rows": int(red[0]), "ranks": world, "bit_exact": bool(mn == 1.0), "max_rel_dev": mx,
              "max_abs_dev": mabs, "tolerance": tol, "passed": passed,
              "rows_spec": "per rank: first and last 1024 rows + every k-th row of its timed batch",
              "oracle": "oracle/obtree_oracle.c evaluate_scalar (full model)"}

    fp16 = None
    if spec.half_leaves and rank == 0 and not plan.reduce:
        fp16 = fp16_report(full_model, x, out, device)

    if graph is not None:
        # per-kernel split from marked stream launches after the timed region
        for m in marks:
            ev.predict_device_marked(x, m, out=out, workspace=ws)
        torch.cuda.synchronize()
    q_ms = sum(m[0].elapsed_ms(m[1]) for m in marks) / len(marks)
    a_ms = sum(m[1].elapsed_ms(m[2]) for m in marks) / len(marks)
    reduce_ms = None
    if plan.reduce:
        # the reduce alone, for the report (it is already inside every timed step above)
        torch.cuda.synchronize()
        t_start.record(stream)
        complete()
        t_end.record(stream)
        torch.cuda.synchronize()
        reduce_ms = t_start.elapsed_ms(t_end)

    # --- end to end through the public API: pinned host features -> scores in pinned host memory
    e2e, e2e_pageable = None, None
    if not args.no_e2e:
        n_e = N if not multi else min(N, args.e2e_multi_objects)
        xh = torch.empty((n_e, spec.n_features), dtype=torch.float32, pin_memory=True)
        xh.copy_(x[:n_e])
        oh = torch.empty((n_e, spec.n_outputs) if multi else n_e, dtype=torch.float64, pin_memory=True)
        fmx = obt.FeatureMatrix(xh.numpy(), obt.Layout.OBJECT_MAJOR)
        ohn = oh.numpy()
        predict_host = sharded.trees.predict if sharded is not None else (lambda m: ev.predict(m, out=ohn))
        predict_host(fmx)
        ke = max(1, min(K, args.e2e_steps))
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(ke):
            predict_host(fmx)
        dt = max_over_ranks(time.perf_counter() - t0, world) / ke
        objs = reduce_over_ranks([n_e], world, "sum")[0] / plan.grid[1]
        e2e = {"value": objs * spec.n_trees / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": n_e * spec.n_features * 4, "d2h_bytes_per_step": n_e * 8 * spec.n_outputs,
               "api": ("TreeShardedEvaluator.predict(FeatureMatrix(pinned numpy)): partials -> NCCL all_reduce -> "
                       "finalize -> host" if sharded is not None else
                       "Evaluator.predict(FeatureMatrix(pinned numpy), out=pinned) -> obt_predict_host"),
               "steps": ke, "objects_per_rank": n_e}
        if n_e < N:
            e2e["sample"] = f"the first {n_e} objects of each rank's batch (host memory bound)"
        del xh, oh
        if world == 1 and not multi and args.e2e_pageable_steps > 0:
            # the literal drop-in call: pageable numpy input, a fresh float64 result
            xp = x.cpu().numpy()
            fmp = obt.FeatureMatrix(xp, obt.Layout.OBJECT_MAJOR)
            ev.predict(fmp)
            kp = args.e2e_pageable_steps
            t0 = time.perf_counter()
            for _ in range(kp):
                ev.predict(fmp)
            dt = (time.perf_counter() - t0) / kp
            e2e_pageable = {"value": N * spec.n_trees / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
                            "h2d_bytes_per_step": N * spec.n_features * 4, "d2h_bytes_per_step": N * 8,
                            "api": "Evaluator.predict(FeatureMatrix(numpy)) -> fresh ndarray (pageable memory)",
                            "steps": kp}
            del xp, fmp

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_port(spec, fm_full, x, spec.n_trees, args.cpu_seconds)
        if not args.no_reference_pkg:
            cpu["reference_pkg"] = reference_pkg_baseline(spec, x, args.cpu_seconds * 4)

    if rank != 0:
        return
    pk = peaks()
    props = torch.cuda.get_device_properties(device)
    n_sm = props.multi_processor_count
    p_int = n_sm * 128 * pk["sm_max_mhz"] * 1e6  # lane-ops/s
    local_spec = synthetic.WorkloadSpec(**{**spec.__dict__, "n_objects": N, "n_trees": te - tb})
    terms = roofline_terms(local_spec)
    apply_achieved = terms["apply_ops"] / (a_ms / 1e3)
    t_roof = max(terms["bytes"] / (pk["hbm_gbs"] * 1e9), terms["ops"] / p_int)
    t_rank = step_s if not plan.reduce else step_s - (reduce_ms or 0) / 1e3
    quant_gbs = terms["quantize_bytes"] / (q_ms / 1e3) / 1e9
    traffic, traffic_src = load_ncu_traffic(args.config)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": plan.scaling, "vs_baseline": None,
        "dtype": "f16/f32" if spec.half_leaves else "f64",
        "data": "synthetic (seeded; BASELINE names no dataset)",
        "config": workload_config(spec, plan, world),
        "device_path": {"n_objects_per_gpu": N, "trees_per_gpu": te - tb,
                        "leaf_storage_on_device": ev.leaf_storage,
                        "quantize_search": quantize_search(ev, spec.n_features),
                        **({"multi_apply": ev.apply_kernel()} if hasattr(ev, "apply_kernel") else {}),
                        "launch": "CUDA graph replay of one predict" if graph is not None else "stream launches",
                        **({"path_options": dict(kv.split("=", 1) for kv in args.path)} if args.path else {})},
        "verify": verify,
        "e2e": e2e,
        "e2e_pageable": e2e_pageable,
        "gpu_launches": launches,
        "roofline": {
            "bound": "issue", "kernel": "tree apply (leaf index + gather + fold)",
            "achieved": apply_achieved / 1e12, "peak": p_int / 1e12, "unit": "Tlane-op/s",
            "frac": apply_achieved / p_int, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_ops_per_launch": terms["apply_ops"], "ms_per_launch": a_ms,
            "ops_definition": "N*T*D split compares + N*T*C leaf gathers (SURVEY.md 8d), per predict",
            "peak_source": f"{n_sm} SMs x 128 lanes x {pk['sm_max_mhz']:.0f} MHz",
        },
        "roofline_step": {"t_roof_ms": t_roof * 1e3, "t_step_ms": t_rank * 1e3, "frac": t_roof / t_rank,
                          "bytes": terms["bytes"], "ops": terms["ops"], "hbm_gbs_peak": pk["hbm_gbs"],
                          "peak_source": pk["source"],
                          "definition": "max(bytes / HBM, ops / integer issue peak) of SURVEY.md 8d over this GPU's "
                                        "share; t_step excludes the collective"},
        "kernels": {"quantize_ms": q_ms, "quantize_GBps": quant_gbs, "quantize_frac_hbm": quant_gbs / pk["hbm_gbs"],
                    "apply_ms": a_ms},
        "clocks": clk,
    }
    if not multi:
        rs = roofline_smem(local_spec, n_sm, pk["sm_max_mhz"] * 1e6, pk["hbm_gbs"], 2 if spec.half_leaves else 4)
        t_floor = (rs["t_apply_floor_ms"] + rs["t_quantize_floor_ms"]) / 1e3
        line["roofline_smem"] = {**rs, "t_floor_ms": t_floor * 1e3, "t_step_ms": t_rank * 1e3,
                                 "frac": t_floor / t_rank, "apply_frac": rs["t_apply_floor_ms"] / a_ms,
                                 "note": "a B200 shared-memory model of this design, secondary to roofline"}
    if plan.reduce:
        line["nccl_reduce_ms"] = reduce_ms
    if fp16 is not None:
        line["fp16_vs_fp32"] = fp16
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def load_ncu_traffic(cfg: int):
    """DRAM bytes per apply launch from the committed ncu capture (not measured in this
    run; the source file is named next to the number)."""
    path = ROOT / "profiles" / "ncu_apply_summary.json"
    if not path.exists():
        return None, None
    try:
        data = json.loads(path.read_text()).get(f"cfg{cfg}", {})
        v = data.get("dram_bytes_per_launch")
        return v, (f"static: {data.get('source', 'profiles/ncu_apply_summary.json')} (committed ncu --set full "
                   "capture, not measured in this run)") if v is not None else None
    except Exception:
        return None, None


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5, 6],
                    help="BASELINE configs 1-5; 6 = the reference bench's epsilon8k64 shape (informational)")
    ap.add_argument("--objects", type=int, default=0, help="override the configuration's object count")
    ap.add_argument("--trees", type=int, default=0, help="override the tree count (experiments)")
    ap.add_argument("--leaves", choices=["fp32", "fp16"], default=None,
                    help="leaf family override: fp16 = binary16 leaves folded in binary32 (config 3 is config 2 + fp16)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="objects: strong = the configuration's batch split over the GPUs (config 4's default), "
                         "weak = one batch of that size per GPU (configs 1-3 default)")
    ap.add_argument("--shard", choices=["objects", "trees", "grid"], default=None,
                    help="config 5: trees (default at N>1), objects, or a 2-D grid (--grid GoxGt)")
    ap.add_argument("--grid", default="1x1")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reference-pkg", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-pageable-steps", type=int, default=2)
    ap.add_argument("--e2e-multi-objects", type=int, default=2_000_000)
    ap.add_argument("--verify-rows", type=int, default=65536)
    ap.add_argument("--ref-sample", type=int, default=65536)
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay a CUDA graph of one predict (auto: when a step is under 0.2 ms)")
    ap.add_argument("--path", action="append", default=[], metavar="NAME=VALUE",
                    help="force a planner choice (obt_set_path_option; A/B runs), e.g. --path desc_source=0")
    ap.add_argument("--refpkg-worker", nargs=5, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.refpkg_worker:
        path, core, offset, n, half = args.refpkg_worker
        refpkg_worker(path, int(core), int(offset), int(n), half == "1")
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    if args.impl == "reference":
        # CPU only, rank 0 only: no process group (the other ranks exit 0 without work)
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup()
    if args.gpus > 1 and world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; running {world} rank(s)", file=sys.stderr)
    try:
        run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
