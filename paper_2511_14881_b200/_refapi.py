"""The reference package's public *types*, when it is importable.

The drop-in replaces the reference's hot-path functions. Callers keep
catching the reference's exceptions (``except filtra.errors.DimMismatch``) and keep
receiving its result types (``filtra.ivf.TopkResult``), because ``except`` and
``isinstance`` match by class, not by name. So when ``filtra`` can be imported in the
running interpreter, the modules of this package re-export the reference's classes in
place of their local look-alikes; otherwise (the GPU box without the reference, or
``FB_REFERENCE_TYPES=0``) the local definitions, which have the same fields,
constructors and messages, stand in. Only class objects are taken from the reference --
no reference code runs on the hot path.
"""

from __future__ import annotations

import importlib
import os


def ref_module(name: str):
    """``filtra.<name>`` or None."""
    if os.environ.get("FB_REFERENCE_TYPES", "1") == "0":
        return None
    try:
        return importlib.import_module(f"filtra.{name}")
    except Exception:  # absent, or a broken install: keep the local types
        return None


def bind(namespace: dict, module: str, names) -> list[str]:
    """Replace ``names`` in ``namespace`` (a module's globals) by the reference's classes of
    the same names, when ``filtra.<module>`` is importable. Returns the names bound."""
    ref = ref_module(module)
    if ref is None:
        return []
    bound = []
    for n in names:
        obj = getattr(ref, n, None)
        if isinstance(obj, type):
            namespace[n] = obj
            bound.append(n)
    return bound
