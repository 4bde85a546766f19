"""Seeded synthetic workloads with the shapes of BASELINE.json's configs.

BASELINE names no public dataset (and the paper's epsilon8k_64 model is not
available), so benches and large parity runs use these generators, following
SURVEY.md section 8(d):

* borders: per-feature quantiles of the feature's distribution, float32;
* splits: per level, feature ~ U{0..F-1}, ordinal ~ U{0..B-1} (the structure of the
  reference generator, synthetic.py:112-122);
* leaves: float32 values ~ N(0, sigma) stored as binary64;
* scale 1, bias 0 (a parity variant draws scale ~ U(0.5, 1.5), bias ~ U(-0.5, 0.5));
* seeds: model 1000*cfg + 1, data 1000*cfg + 2.

Models are vectorised numpy draws (np.random.default_rng); features for the small
configs come from numpy on the host, for the large ones from a CUDA torch.Generator
directly in HBM (64 GB at config 5 cannot be staged from the host).
"""

from __future__ import annotations

from dataclasses import dataclass
from statistics import NormalDist

import numpy as np

from .model import FloatFeatureBorders, ObliviousModel, ObliviousTree, SplitCondition

NORMAL, UNIFORM100, LOGNORMAL, INT1000 = "normal", "uniform100", "lognormal", "int1000"


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    n_objects: int
    n_features: int
    borders: int
    n_trees: int
    depth: int
    leaf_sigma: float
    n_outputs: int = 1
    half_leaves: bool = False
    cfg: int = 0

    def feature_kind(self, f: int) -> str:
        if self.cfg == 2 or self.cfg == 3:
            return NORMAL if f < self.n_features // 2 else UNIFORM100
        if self.cfg == 4:
            return (NORMAL, LOGNORMAL, INT1000)[f % 3]
        return NORMAL

    @property
    def model_seed(self) -> int:
        return 1000 * self.cfg + 1

    @property
    def data_seed(self) -> int:
        return 1000 * self.cfg + 2


CONFIGS = {
    1: WorkloadSpec("cfg1-10k-f50-b16-t500-d6", 10_000, 50, 16, 500, 6, 0.1, cfg=1),
    2: WorkloadSpec("cfg2-1m-f200-b64-t2000-d6", 1_000_000, 200, 64, 2000, 6, 0.05, cfg=2),
    3: WorkloadSpec("cfg3-1m-f200-b64-t2000-d6-fp16", 1_000_000, 200, 64, 2000, 6, 0.05, half_leaves=True, cfg=3),
    4: WorkloadSpec("cfg4-8m-f500-b128-t8000-d8", 8_000_000, 500, 128, 8000, 8, 0.02, cfg=4),
    5: WorkloadSpec("cfg5-16m-f1000-b254-t4000-d10-c10", 16_000_000, 1000, 254, 4000, 10, 0.01, n_outputs=10, cfg=5),
    # informational (not a BASELINE config): the shape of the reference bench's
    # "epsilon8k64" preset -- the paper's published single-core model, 2,000 features,
    # 64 borders, 8,000 depth-6 trees (reference bench.py:40-44) -- on 1M N(0,1) objects
    6: WorkloadSpec("eps8k64-1m-f2000-b64-t8000-d6", 1_000_000, 2000, 64, 8000, 6, 0.05, cfg=6),
}


def quantile_borders(kind: str, count: int) -> np.ndarray:
    """Border k = float32 quantile (k+1)/(B+1) of the feature's distribution."""
    p = [(k + 1) / (count + 1) for k in range(count)]
    nd = NormalDist()
    if kind == NORMAL:
        vals = [nd.inv_cdf(q) for q in p]
    elif kind == UNIFORM100:
        vals = [100.0 * q for q in p]
    elif kind == LOGNORMAL:
        vals = [float(np.exp(nd.inv_cdf(q))) for q in p]
    elif kind == INT1000:
        vals = [float(int(1000 * (k + 1) // (count + 1))) for k in range(count)]
    else:
        raise ValueError(kind)
    out = np.array(vals, dtype=np.float32)
    if count > 1 and not np.all(np.diff(out) > 0):
        raise ValueError(f"{kind} borders collide at float32 for B={count}")
    return out


def model_arrays(spec: WorkloadSpec, seed=None, affine: bool = False) -> dict:
    """Flat arrays of the synthetic model (leaves [T][C][2^D] float64)."""
    rng = np.random.default_rng(spec.model_seed if seed is None else seed)
    borders = [quantile_borders(spec.feature_kind(f), spec.borders) for f in range(spec.n_features)]
    shape = (spec.n_trees, spec.depth)
    split_feature = rng.integers(0, spec.n_features, size=shape, dtype=np.int64).astype(np.int32)
    split_ordinal = rng.integers(0, spec.borders, size=shape, dtype=np.int64).astype(np.int32)
    leaves = rng.normal(0.0, spec.leaf_sigma, size=(spec.n_trees, spec.n_outputs, 1 << spec.depth))
    leaves = leaves.astype(np.float32).astype(np.float64)
    scale, bias = 1.0, 0.0
    if affine:
        scale = float(rng.uniform(0.5, 1.5))
        bias = float(rng.uniform(-0.5, 0.5))
    return {
        "borders": borders,
        "split_feature": split_feature,
        "split_ordinal": split_ordinal,
        "leaves": leaves,
        "scale": scale,
        "bias": bias,
    }


def build_model(spec: WorkloadSpec, seed=None, affine: bool = False) -> ObliviousModel:
    """The synthetic single-output model as reference-compatible types."""
    if spec.n_outputs != 1:
        raise ValueError("ObliviousModel holds one output; use model_arrays for multiclass")
    a = model_arrays(spec, seed, affine)
    feats = tuple(FloatFeatureBorders(f, b) for f, b in enumerate(a["borders"]))
    trees = tuple(
        ObliviousTree(
            depth=spec.depth,
            splits=tuple(SplitCondition(int(f), int(o)) for f, o in zip(a["split_feature"][t], a["split_ordinal"][t])),
            leaf_values=a["leaves"][t, 0],
        )
        for t in range(spec.n_trees)
    )
    return ObliviousModel(float_features=feats, trees=trees, scale=a["scale"], bias=a["bias"])


def host_features(spec: WorkloadSpec, n_objects=None, seed=None) -> np.ndarray:
    """Object-major float32 [n][F] drawn on the host (configs 1-3 and samples)."""
    n = spec.n_objects if n_objects is None else n_objects
    rng = np.random.default_rng(spec.data_seed if seed is None else seed)
    x = np.empty((n, spec.n_features), dtype=np.float32)
    kinds = [spec.feature_kind(f) for f in range(spec.n_features)]
    for kind in sorted(set(kinds)):
        cols = np.array([f for f, k in enumerate(kinds) if k == kind])
        x[:, cols] = _draw(rng, kind, (n, cols.size))
    return x


def _draw(rng, kind: str, shape) -> np.ndarray:
    if kind == NORMAL:
        return rng.standard_normal(shape, dtype=np.float32)
    if kind == UNIFORM100:
        return (rng.random(shape, dtype=np.float32) * np.float32(100.0)).astype(np.float32)
    if kind == LOGNORMAL:
        return np.exp(rng.standard_normal(shape, dtype=np.float32)).astype(np.float32)
    if kind == INT1000:
        return rng.integers(0, 1001, size=shape).astype(np.float32)
    raise ValueError(kind)


def device_features(spec: WorkloadSpec, n_objects=None, seed=None, device="cuda"):
    """Object-major float32 [n][F] generated in HBM with a seeded CUDA generator."""
    import torch

    n = spec.n_objects if n_objects is None else n_objects
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.data_seed if seed is None else seed)
    x = torch.empty((n, spec.n_features), dtype=torch.float32, device=device)
    kinds = [spec.feature_kind(f) for f in range(spec.n_features)]
    if all(k == NORMAL for k in kinds):
        x.normal_(generator=gen)
        return x
    for kind in sorted(set(kinds)):
        cols = torch.tensor([f for f, k in enumerate(kinds) if k == kind], device=device)
        shape = (n, int(cols.numel()))
        if kind == NORMAL:
            block = torch.randn(shape, generator=gen, device=device)
        elif kind == UNIFORM100:
            block = torch.rand(shape, generator=gen, device=device) * 100.0
        elif kind == LOGNORMAL:
            block = torch.randn(shape, generator=gen, device=device).exp_()
        else:
            block = torch.randint(0, 1001, shape, generator=gen, device=device).float()
        x.index_copy_(1, cols, block)
        del block
    return x


def sprinkle_specials(x: np.ndarray, borders, seed: int, nan=0.02, inf=0.01, exact=0.02, denorm=0.01) -> np.ndarray:
    """Parity variant: NaN / +-inf / exact-border hits / denormals at the given rates
    (test_acceptance.py:112-115 rates for NaN and inf)."""
    rng = np.random.default_rng(seed)
    x = x.copy()
    n, F = x.shape
    roll = rng.random((n, F))
    x[roll < nan] = np.nan
    infs = (roll >= nan) & (roll < nan + inf)
    x[infs] = np.where(rng.random(int(infs.sum())) < 0.5, np.inf, -np.inf).astype(np.float32)
    ex = (roll >= nan + inf) & (roll < nan + inf + exact)
    rows, cols = np.nonzero(ex)
    for r, c in zip(rows, cols):
        b = borders[c]
        if b.size:
            x[r, c] = b[rng.integers(0, b.size)]
    dn = (roll >= nan + inf + exact) & (roll < nan + inf + exact + denorm)
    tiny = (rng.random(int(dn.sum())) * 2.0**-130).astype(np.float32)
    x[dn] = np.where(rng.random(tiny.size) < 0.5, tiny, -tiny)
    return x
