"""Small host<->device helpers (torch is the allocator/stream provider only)."""

from __future__ import annotations

import numpy as np
import torch


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def to_dev_u64(a, dev=None) -> torch.Tensor:
    """uint64 data (numpy or torch) -> int64-typed CUDA tensor holding the same bits."""
    dev = dev or device()
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.uint64:
            a = a.view(torch.int64)
        return a.to(dev).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint64)).view(np.int64)
    return torch.from_numpy(arr.copy()).to(dev)


def to_dev(a, dtype, dev=None) -> torch.Tensor:
    dev = dev or device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype).contiguous()


def u64_host(t: torch.Tensor) -> np.ndarray:
    """int64-typed tensor holding uint64 bits -> numpy uint64."""
    return t.detach().cpu().numpy().view(np.uint64)


def pad_rows_i8(items: torch.Tensor, dim_pad: int, n_rows: int) -> torch.Tensor:
    """int8 [n, dim] -> zero-padded int8 [n_rows, dim_pad] on the same device."""
    out = torch.zeros((n_rows, dim_pad), dtype=torch.int8, device=items.device)
    out[: items.shape[0], : items.shape[1]] = items
    return out


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m
