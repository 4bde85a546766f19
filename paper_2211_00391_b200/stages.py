"""Stage-level GPU entry points, for parity checks and debugging.

``quantize`` runs stage 1 alone (reference quantize_block, quantize.py:136-172) and
returns the reference's bucket ids; ``leaf_indices`` runs the same quantize +
index code the predict path runs (reference compute_leaf_indices / _leaf_index_panel,
indexer.py:39-57, evaluate.py:199-207) and returns the per-tree leaf indices.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .evaluate import ModelTables
from .matrix import Layout, layout_code
from .model import LeafPrecision


def _prepare(model_or_tables, x, layout: Layout):
    import torch

    tables = model_or_tables if isinstance(model_or_tables, ModelTables) else ModelTables(model_or_tables)
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32 and x.dim() == 2):
        raise TypeError("expected a 2-D float32 CUDA tensor")
    x = x.contiguous()
    n, f = (x.shape[0], x.shape[1]) if layout is Layout.OBJECT_MAJOR else (x.shape[1], x.shape[0])
    if f != tables.n_features:
        raise ValueError(f"matrix has {f} features, model expects {tables.n_features}")
    dev = tables.device_model(LeafPrecision.BINARY64, x.device.index or 0)
    return tables, dev, x, n


def quantize(model_or_tables, x, layout: Layout = Layout.OBJECT_MAJOR):
    """uint8 CUDA tensor [F][n]: bucket = #{k : x > border_k}, NaN -> 0."""
    import torch

    tables, dev, x, n = _prepare(model_or_tables, x, layout)
    out = torch.empty((tables.n_features, n), dtype=torch.uint8, device=x.device)
    if n:
        stream = _native.current_stream_handle(x.device)
        _native.check(dev._lib.obt_quantize_dev(dev.handle, x.data_ptr(), n, layout_code(layout), out.data_ptr(), stream))
    return out


def leaf_indices(model_or_tables, x, layout: Layout = Layout.OBJECT_MAJOR, tree_begin: int = 0, tree_end=None):
    """int16 CUDA tensor [trees][n] holding the uint16 leaf index of every (tree, object)."""
    import torch

    tables, dev, x, n = _prepare(model_or_tables, x, layout)
    tree_end = tables.n_trees if tree_end is None else tree_end
    out = torch.empty((max(0, tree_end - tree_begin), n), dtype=torch.int16, device=x.device)
    stream = _native.current_stream_handle(x.device)
    _native.check(
        dev._lib.obt_leaf_indices_dev(
            dev.handle, x.data_ptr(), n, layout_code(layout), int(tree_begin), int(tree_end), out.data_ptr(), stream
        )
    )
    return out


def as_uint16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)
