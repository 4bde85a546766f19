"""Argument checks shared by every predict entry point (host and device).

The kernels write n (or n x C) float64 values through the raw output pointer and use
the workspace pointer as scratch, so every buffer a caller supplies is checked here
before a pointer reaches the C ABI: dtype, shape, contiguity and device.  The texts
of the feature-count error are the reference's (evaluate.py:271-274).
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .matrix import Layout


def check_features(matrix_features: int, model_features: int) -> None:
    if matrix_features != model_features:
        raise ValueError(f"matrix has {matrix_features} features, model expects {model_features}")


def out_shape(n: int, n_outputs: int) -> tuple:
    return (n,) if n_outputs == 1 else (n, n_outputs)


def host_out(out: Optional[np.ndarray], n: int, n_outputs: int) -> np.ndarray:
    """A fresh float64 result, or the caller's ``out`` after checking it can hold one."""
    shape = out_shape(n, n_outputs)
    if out is None:
        return np.empty(shape, dtype=np.float64)
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != shape or not out.flags.c_contiguous:
        raise ValueError(f"out must be a contiguous float64 array of shape {shape}")
    if not out.flags.writeable:
        raise ValueError("out must be writeable")
    return out


def device_inputs(x, layout: Layout, model_features: int, device: int, n_outputs: int = 1, out=None,
                  workspace=None):
    """Validated (x, n, out, ws_ptr, ws_bytes) for a device predict.

    ``x``: 2-D float32 CUDA tensor on the model's device ([n][F] object-major or [F][n]
    feature-major; made contiguous).  ``out``: float64 CUDA tensor of shape (n,) or
    (n, C), contiguous, on the same device (allocated when None).  ``workspace``: uint8
    CUDA tensor on the same device (or None: the library's pool)."""
    import torch

    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise TypeError("predict_device expects a CUDA tensor")
    if x.dtype != torch.float32 or x.dim() != 2:
        raise ValueError("feature tensor must be 2-D float32")
    if x.device.index != device:
        raise ValueError(f"feature tensor is on cuda:{x.device.index}, the model on cuda:{device}")
    x = x.contiguous()
    n, f = (x.shape[0], x.shape[1]) if layout is Layout.OBJECT_MAJOR else (x.shape[1], x.shape[0])
    check_features(f, model_features)
    shape = out_shape(n, n_outputs)
    if out is None:
        out = torch.empty(shape, dtype=torch.float64, device=x.device)
    elif not (isinstance(out, torch.Tensor) and out.is_cuda and out.device == x.device
              and out.dtype == torch.float64 and tuple(out.shape) == shape and out.is_contiguous()):
        raise ValueError(f"out must be a contiguous float64 CUDA tensor of shape {shape} on {x.device}")
    ws_ptr, ws_bytes = 0, 0
    if workspace is not None:
        if not (isinstance(workspace, torch.Tensor) and workspace.is_cuda and workspace.device == x.device
                and workspace.dtype == torch.uint8 and workspace.is_contiguous()):
            raise ValueError(f"workspace must be a contiguous uint8 CUDA tensor on {x.device}")
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel()
    return x, n, out, ws_ptr, ws_bytes
