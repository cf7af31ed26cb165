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


class IdentityCache:
    """Values keyed on an object's IDENTITY, dropped when the object is collected.

    The reference's engine parts (``IvfIndex``, ``BloomIndex``, ``EmbeddingCache``, the
    scorers) are ``@dataclass`` instances: ``eq=True`` makes them unhashable, so a
    ``WeakKeyDictionary`` cannot hold them and every request would re-upload them. Entries
    here hold a weak reference (the value dies with its host object, so a snapshot hot swap
    frees the old device copy); objects that cannot be weakly referenced are held strongly,
    at most ``max_strong`` of them (LRU)."""

    def __init__(self, max_strong: int = 8):
        import threading
        from collections import OrderedDict
        self._d: dict = {}
        self._strong: "OrderedDict" = OrderedDict()
        self._max_strong = max_strong
        self._lock = threading.Lock()

    def get(self, obj):
        with self._lock:
            e = self._d.get(id(obj))
            if e is None:
                return None
            ref, val = e
            if ref is None:  # strongly held
                if self._strong.get(id(obj)) is not obj:
                    return None
                self._strong.move_to_end(id(obj))
                return val
            return val if ref() is obj else None

    def put(self, obj, val) -> None:
        import weakref
        k = id(obj)

        def drop(r, k=k):
            with self._lock:
                e = self._d.get(k)
                if e is not None and e[0] is r:
                    del self._d[k]

        try:
            ref = weakref.ref(obj, drop)
        except TypeError:
            ref = None
        with self._lock:
            self._d[k] = (ref, val)
            if ref is None:
                self._strong[k] = obj
                self._strong.move_to_end(k)
                while len(self._strong) > self._max_strong:
                    old, _ = self._strong.popitem(last=False)
                    self._d.pop(old, None)

    def get_or_make(self, obj, make):
        hit = self.get(obj)
        if hit is None:
            hit = make(obj)
            self.put(obj, hit)
        return hit
