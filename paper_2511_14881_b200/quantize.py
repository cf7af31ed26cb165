"""Global min/max int8 quantisation (reference quantize.py:1-102).

One affine map for items and queries: ``clip(rint((x - min) * 255/(max-min)) - 128,
-128, 127)`` in float64 with round-half-to-even -- computed by the ``fb_quantize``
kernel with ``__dsub_rn``/``__dmul_rn`` (no contraction), so codes are bit-identical
to NumPy's. Exact int32 dots run on the device (``fb_int8_dot_rows``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import device, to_dev
from .errors import DegenerateRange, LengthMismatch


@dataclass(frozen=True)
class QuantParams:
    global_min: float
    global_max: float

    @property
    def scale(self) -> float:
        return 255.0 / (self.global_max - self.global_min)

    @property
    def step(self) -> float:
        return (self.global_max - self.global_min) / 255.0


@dataclass(frozen=True)
class QuantizedMatrix:
    data: np.ndarray
    params: QuantParams


def compute_quant_params(matrix) -> QuantParams:
    """Global min and max over all cells (reference quantize.py:41-55)."""
    if isinstance(matrix, torch.Tensor):
        if matrix.numel() == 0:
            raise DegenerateRange("empty matrix")
        lo, hi = float(matrix.min()), float(matrix.max())
    else:
        matrix = np.asarray(matrix)
        if matrix.size == 0:
            raise DegenerateRange("empty matrix")
        lo, hi = float(matrix.min()), float(matrix.max())
    if lo == hi or not np.isfinite(255.0 / (hi - lo)):
        raise DegenerateRange(f"cells span degenerate range [{lo}, {hi}]")
    return QuantParams(global_min=lo, global_max=hi)


def quantize_device(x: torch.Tensor, params: QuantParams, out_stride: int | None = None,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """float32/float64 CUDA [rows, cols] -> int8 CUDA [rows, out_stride] (zero-padded
    columns)."""
    lib = _native.lib()
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    x = x.to(device=device()).contiguous()
    if x.dim() == 1:
        x = x.view(1, -1)
    rows, cols = x.shape
    stride = out_stride if out_stride is not None else cols
    if out is None:
        out = torch.empty((rows, stride), dtype=torch.int8, device=x.device)
    fn = lib.fb_quantize if x.dtype == torch.float32 else lib.fb_quantize_f64
    _native.check(fn(x.data_ptr(), rows, cols, float(params.global_min),
                     float(params.global_max), out.data_ptr(), stride, _native.stream_ptr()))
    return out


def quantize_value(x: float, params: QuantParams) -> int:
    return int(quantize_vector(np.array([x], dtype=np.float64), params)[0])


def quantize_matrix(matrix, params: QuantParams) -> QuantizedMatrix:
    m = np.asarray(matrix)
    q = _quantize_host_roundtrip(m.reshape(-1, m.shape[-1]) if m.ndim > 1 else m.reshape(1, -1),
                                 params)
    return QuantizedMatrix(data=q.reshape(m.shape), params=params)


def quantize_vector(vec, params: QuantParams) -> np.ndarray:
    """reference quantize.py:72-76, computed on the GPU."""
    v = np.asarray(vec)
    return _quantize_host_roundtrip(v.reshape(1, -1), params).reshape(v.shape)


def _quantize_host_roundtrip(m: np.ndarray, params: QuantParams) -> np.ndarray:
    dt = torch.float32 if m.dtype == np.float32 else torch.float64
    x = to_dev(m.astype(np.float32 if dt == torch.float32 else np.float64), dt)
    return quantize_device(x, params).cpu().numpy()


def dequantize(q, params: QuantParams):
    """Bucket-centre floats (reference quantize.py:79-81); host helper."""
    return (np.asarray(q, dtype=np.float64) + 128.0) / params.scale + params.global_min


def int8_dot_rows(rows, vec) -> np.ndarray:
    """Exact int32 dot of each int8 row with an int8 vector (reference quantize.py:96-102)."""
    rows = np.asarray(rows, dtype=np.int8)
    vec = np.asarray(vec, dtype=np.int8)
    if rows.shape[-1] != vec.shape[0]:
        raise LengthMismatch(rows.shape[-1], vec.shape[0])
    r2 = rows.reshape(-1, rows.shape[-1])
    lib = _native.lib()
    dev = device()
    rt = to_dev(r2, torch.int8, dev)
    vt = to_dev(vec, torch.int8, dev)
    out = torch.empty(r2.shape[0], dtype=torch.int32, device=dev)
    _native.check(lib.fb_int8_dot_rows(rt.data_ptr(), r2.shape[0], r2.shape[1], r2.shape[1],
                                       vt.data_ptr(), out.data_ptr(), _native.stream_ptr()))
    return out.cpu().numpy().reshape(rows.shape[:-1])


def int8_dot(a, b) -> int:
    """Exact sum a_i b_i in int32 (reference quantize.py:84-93)."""
    a = np.asarray(a, dtype=np.int8)
    b = np.asarray(b, dtype=np.int8)
    if a.shape != b.shape:
        raise LengthMismatch(a.size, b.size)
    return int(int8_dot_rows(a.reshape(1, -1), b)[0])

