#!/usr/bin/env python
"""Benchmark: object-trees/s of oblivious-ensemble predict on B200, with roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One "step" is one predict over one batch of the workload (BASELINE.json configs[1]
by default: 1,000,000 objects x 200 features, 64 borders, 2,000 depth-6 trees, fp32
leaves).  Under torchrun each rank owns one GPU and its own batch of that size
(object sharding, no data-path collective: weak scaling); NCCL carries only the
barrier and the max-over-ranks of the device-timed region.

Printed on rank 0 as ONE JSON line:
  value      whole-job object-trees/s, features resident in HBM, CUDA-event timed
  e2e        the same metric through Evaluator.predict with pinned host buffers
             (host->device features and device->host scores inside the timed region)
  roofline   the dominant kernel (tree apply) against the integer-issue peak, plus the
             whole-step roofline of BASELINE.md section 6
  cpu_baseline  the C oracle port of the reference algorithm on this host's cores
`--impl reference` times that CPU port alone on the same config and metric.
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


def cpu_baseline(spec, model, seconds: float, verify_fn=None) -> dict:
    """The C oracle port of the reference algorithm on this host's cores, on a bounded
    prefix sample of the same workload (doubling until the run takes >= `seconds`/4)."""
    import numpy as np

    import oracle
    from paper_2211_00391_b200 import synthetic

    fm = flat_model(model)
    oracle.set_threads(oracle.host_cores())  # all host cores, whatever OMP_NUM_THREADS says
    threads = oracle.max_threads()
    n = 4096
    best = None
    while True:
        x = synthetic.host_features(spec, n_objects=n, seed=spec.data_seed + 7)
        t0 = time.perf_counter()
        ref = oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR,
                                     oracle.BINARY16 if spec.half_leaves else oracle.BINARY64)
        dt = time.perf_counter() - t0
        best = (n, dt, x, ref)
        if dt >= seconds / 4 or n >= spec.n_objects or n >= 1 << 22:
            break
        n *= 2
    n, dt, x, ref = best
    reps = max(1, int(round(seconds * 0.75 / max(dt, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.evaluate_scalar(fm, x, oracle.OBJECT_MAJOR, oracle.BINARY16 if spec.half_leaves else oracle.BINARY64)
    dt = (time.perf_counter() - t0) / reps
    out = {
        "value": n * spec.n_trees / dt,
        "unit": UNIT,
        "cores": threads,
        "host_cpus": os.cpu_count(),
        "kind": "port",
        "sample": f"first {n} objects of the workload (full {spec.n_trees}-tree model), {reps} reps, "
                  f"C restatement of evaluate_scalar (oracle/obtree_oracle.c), OpenMP over objects",
    }
    if verify_fn is not None:
        got = verify_fn(x)
        out["gpu_verified_bit_exact"] = bool(np.array_equal(got, ref))
        rel = np.abs(got - ref) / np.maximum(np.maximum(np.abs(got), np.abs(ref)), 1e-300)
        out["gpu_max_rel_dev"] = float(rel.max()) if rel.size else 0.0
    return out


def load_ncu_mio(cfg: int):
    """The dominant kernel's shared-memory wavefront rate as a fraction of peak (ncu), the
    resource that binds this path on B200."""
    path = ROOT / "profiles" / "ncu_apply_summary.json"
    if not path.exists():
        return None
    try:
        v = json.loads(path.read_text()).get(f"cfg{cfg}", {}).get("smem_wavefront_pct_of_peak")
        return None if v is None else v / 100.0
    except Exception:
        return None


def load_ncu_traffic(cfg: int):
    path = ROOT / "profiles" / "ncu_apply_summary.json"
    if not path.exists():
        return None
    try:
        data = json.loads(path.read_text())
        return data.get(f"cfg{cfg}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_reference(args, world, rank):
    """--impl reference: the CPU port of the reference algorithm, all host threads."""
    if rank != 0:
        return
    import numpy as np  # noqa: F401

    import oracle
    from paper_2211_00391_b200 import synthetic

    spec = synthetic.CONFIGS[args.config]
    if spec.n_outputs > 1:
        from paper_2211_00391_b200 import multiclass

        model = multiclass.from_arrays(synthetic.model_arrays(spec))
    else:
        model = synthetic.build_model(spec)
    fm = flat_model(model)
    oracle.set_threads(oracle.host_cores())  # torchrun exports OMP_NUM_THREADS=1; use every core
    prec = oracle.BINARY16 if spec.half_leaves else oracle.BINARY64
    n = args.ref_sample
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
        "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16/f32" if spec.half_leaves else "f64", "data": "synthetic",
        "config": {"workload": spec.name, "n_objects_per_step": n, "features": spec.n_features,
                   "borders": spec.borders, "trees": spec.n_trees, "depth": spec.depth},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.max_threads(), "host_cpus": os.cpu_count(),
                         "kind": "port",
                         "sample": f"{n} objects per step of {spec.name}; the reference is pure Python/numpy and "
                                   f"cannot travel, so its algorithm runs as the C oracle port"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_2211_00391_b200 as obt
    from paper_2211_00391_b200 import _native, synthetic

    spec = synthetic.CONFIGS[args.config]
    if args.objects:
        spec = synthetic.WorkloadSpec(**{**spec.__dict__, "n_objects": args.objects})
    if args.trees:
        spec = synthetic.WorkloadSpec(**{**spec.__dict__, "n_trees": args.trees})
    device = local
    torch.cuda.set_device(device)
    multi = spec.n_outputs > 1
    if multi:
        # config 5: tree-sharded across ranks (each rank folds its trees for all objects,
        # partial sums reduced after the timed region); at N=1 the whole model
        from paper_2211_00391_b200 import multiclass, sharding

        full_model = multiclass.from_arrays(synthetic.model_arrays(spec))
        tb, te = sharding.tree_shard(full_model.n_trees, rank, world)
        model = full_model.subset(tb, te, raw=world > 1) if world > 1 else full_model
        ev = multiclass.MultiOutputEvaluator(model, device=device)
    else:
        model = synthetic.build_model(spec)
        strategy = obt.LeafStrategy.NAIVE16 if spec.half_leaves else obt.LeafStrategy.NAIVE
        ev = obt.Evaluator(model, obt.EvalConfig(strategy=strategy), device=device)
    data_seed = spec.data_seed + (0 if multi else 1000 * rank)  # tree sharding: same objects on every rank
    x = synthetic.device_features(spec, seed=data_seed, device=f"cuda:{device}")
    N = spec.n_objects
    out = torch.empty((N, spec.n_outputs) if multi else N, dtype=torch.float64, device=x.device)
    ws = torch.empty(ev.workspace_bytes(N), dtype=torch.uint8, device=x.device)

    tree_sharded = multi and world > 1

    def reduce_partials():
        # tree sharding: a prediction is complete only after the NCCL sum of the ranks'
        # binary64 partial sums and the affine finalize, so both are part of every step
        import torch.distributed as dist

        red = out if reduce_device() == "cuda" else out.cpu()
        dist.all_reduce(red, op=dist.ReduceOp.SUM)
        if red is not out:
            out.copy_(red)
        out.mul_(full_model.scale).add_(full_model.bias)

    for _ in range(args.warmup):
        ev.predict_device(x, out=out, workspace=ws)
        if tree_sharded:
            reduce_partials()
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
    use_graph = not tree_sharded and (args.graph == "on" or (args.graph == "auto" and one_ms < 0.2))
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
        if tree_sharded:
            reduce_partials()
    t_end.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier(world)
    clk = clocks.stop(w0, w1)
    elapsed_ms = max_over_ranks(t_start.elapsed_ms(t_end), world)
    if graph is not None:
        # per-kernel split from marked stream launches after the timed region
        for m in marks:
            ev.predict_device_marked(x, m, out=out, workspace=ws)
        torch.cuda.synchronize()
    q_ms = sum(m[0].elapsed_ms(m[1]) for m in marks) / len(marks)
    a_ms = sum(m[1].elapsed_ms(m[2]) for m in marks) / len(marks)
    step_s = elapsed_ms / K / 1e3
    # object sharding: every rank folds all trees for its own N objects; tree sharding
    # (config 5): every rank folds its share of the trees for the same N objects
    value = (N * spec.n_trees if multi else world * N * spec.n_trees) / step_s
    reduce_ms = None
    if tree_sharded:
        # the reduce alone, for the report (it is already inside every timed step above)
        torch.cuda.synchronize()
        r0 = time.perf_counter()
        reduce_partials()
        torch.cuda.synchronize()
        reduce_ms = (time.perf_counter() - r0) * 1e3

    # end to end through the public API: pinned host features -> scores in pinned host memory
    e2e = None
    if not args.no_e2e and not multi:
        xh = torch.empty((N, spec.n_features), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        oh = torch.empty(N, dtype=torch.float64, pin_memory=True)
        fmx = obt.FeatureMatrix(xh.numpy(), obt.Layout.OBJECT_MAJOR)
        ohn = oh.numpy()
        ev.predict(fmx, out=ohn)
        ke = max(1, min(K, args.e2e_steps))
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(ke):
            ev.predict(fmx, out=ohn)
        dt = max_over_ranks(time.perf_counter() - t0, world) / ke
        e2e = {"value": world * N * spec.n_trees / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": N * spec.n_features * 4, "d2h_bytes_per_step": N * 8,
               "api": "Evaluator.predict(FeatureMatrix, out=pinned) -> obt_predict_host", "steps": ke}
        del xh, oh

    if rank != 0:
        return
    pk = peaks()
    import ctypes

    sms = ctypes.c_int()
    props = torch.cuda.get_device_properties(device)
    n_sm = props.multi_processor_count
    p_int = n_sm * 128 * pk["sm_max_mhz"] * 1e6  # lane-ops/s
    terms = roofline_terms(spec)
    apply_achieved = terms["apply_ops"] / (a_ms / 1e3)
    t_roof = max(terms["bytes"] / (pk["hbm_gbs"] * 1e9), terms["ops"] / p_int)
    quant_gbs = terms["quantize_bytes"] / (q_ms / 1e3) / 1e9

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16/f32" if spec.half_leaves else "f64",
        "data": "synthetic (seeded; BASELINE names no dataset)",
        "config": {"workload": spec.name, "n_objects_per_gpu": N, "features": spec.n_features,
                   "borders": spec.borders, "trees": spec.n_trees, "depth": spec.depth,
                   "leaves": "fp16 (binary32 fold)" if spec.half_leaves else "fp32 values (binary64 fold)",
                   "leaf_storage_on_device": ev.leaf_storage,
                   "quantize_search": quantize_search(ev, spec.n_features),
                   **({"multi_apply": ev.apply_kernel()} if hasattr(ev, "apply_kernel") else {}),
                   "l2": ("inputs larger than L2 (features 4NF bytes, buckets NF bytes > 126 MB)"
                          if 4 * N * spec.n_features > 126e6 else
                          "inputs L2-resident between steps (features 4NF bytes < 126 MB; a launch-bound size)"),
                   "parallelism": f"objects sharded over {world} GPU(s), no data-path collective",
                   "launch": "CUDA graph replay of one predict" if graph is not None else "stream launches"},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {
            "bound": "issue", "kernel": "apply_kernel (leaf index + gather + fold)",
            "achieved": apply_achieved / 1e12, "peak": p_int / 1e12, "unit": "Tlane-op/s",
            "frac": apply_achieved / p_int, "traffic": load_ncu_traffic(args.config),
            "binding_resource": {"what": "shared-memory wavefronts (one 128-byte wavefront per SM per clock)",
                                 "frac_of_peak_ncu": load_ncu_mio(args.config)},
            "algorithmic_ops_per_launch": terms["apply_ops"], "ms_per_launch": a_ms,
            "ops_definition": "N*T*D split compares + N*T*C leaf gathers (SURVEY.md 8d)",
            "peak_source": f"{n_sm} SMs x 128 lanes x {pk['sm_max_mhz']:.0f} MHz",
        },
        "roofline_step": {"t_roof_ms": t_roof * 1e3, "t_step_ms": step_s * 1e3, "frac": t_roof / step_s,
                          "bytes": terms["bytes"], "ops": terms["ops"], "hbm_gbs_peak": pk["hbm_gbs"],
                          "peak_source": pk["source"]},
        "kernels": {"quantize_ms": q_ms, "quantize_GBps": quant_gbs, "quantize_frac_hbm": quant_gbs / pk["hbm_gbs"],
                    "apply_ms": a_ms},
        "clocks": clk,
    }
    if not multi:
        rs = roofline_smem(spec, n_sm, pk["sm_max_mhz"] * 1e6, pk["hbm_gbs"], 2 if spec.half_leaves else 4)
        t_floor = (rs["t_apply_floor_ms"] + rs["t_quantize_floor_ms"]) / 1e3
        line["roofline_smem"] = {**rs, "t_floor_ms": t_floor * 1e3, "t_step_ms": step_s * 1e3, "frac": t_floor / step_s,
                                 "apply_frac": rs["t_apply_floor_ms"] / a_ms}
    if multi:
        line["config"]["outputs"] = spec.n_outputs
        line["config"]["parallelism"] = (f"trees sharded over {world} GPU(s); NCCL all_reduce of fp64 partials "
                                         "+ finalize inside every timed step")
        line["scaling"] = "strong"
        line["nccl_reduce_ms"] = reduce_ms
    if world == 1 and not args.no_cpu_baseline:
        def verify(xs):
            return ev.predict(obt.FeatureMatrix(xs, obt.Layout.OBJECT_MAJOR))

        line["cpu_baseline"] = cpu_baseline(spec, model, args.cpu_seconds, verify)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--objects", type=int, default=0, help="override objects per GPU")
    ap.add_argument("--trees", type=int, default=0, help="override the tree count (experiments)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ref-sample", type=int, default=65536)
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay a CUDA graph of one predict (auto: when a step is under 0.2 ms)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup()
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
