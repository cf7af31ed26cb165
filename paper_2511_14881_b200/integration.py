"""Switch a running reference ``filtra`` installation to the B200 hot path.

``install()`` is INTEGRATION.md's monkey-patch recipe as code: every reference hot-path
function listed in ``PATCHES`` is replaced by this package's
same-signature drop-in -- in its defining module AND in every other ``filtra.*`` module
that bound it by ``from .x import f`` -- so the reference's own callers (``retrieve``,
``sharded_retrieve``, ``handle_batch``, the CLI) and its own tests run on the GPU
unchanged. ``uninstall(record)`` restores the originals.

The result / counter / exception types need no patching: when ``filtra`` is importable
this package already raises and returns the reference's own classes (``_refapi``).
"""

from __future__ import annotations

import importlib
import pkgutil
import sys

from . import bloom, filter_query, ivf, overarch, quantize, retrieval, serve

# (reference module, function name, drop-in) -- reference file:line of each original
PATCHES = [
    ("bloom", "hash_positions", bloom.hash_positions),            # ref/bloom.py:86
    ("bloom", "build_bloom", bloom.build_bloom),                  # ref/bloom.py:114
    ("bloom", "bloom_eval_leaf", bloom.bloom_eval_leaf),          # ref/bloom.py:160
    ("filter_query", "eval_compiled", filter_query.eval_compiled),  # ref/filter_query.py:314
    ("quantize", "quantize_vector", quantize.quantize_vector),    # ref/quantize.py:72
    ("quantize", "int8_dot", quantize.int8_dot),                  # ref/quantize.py:84
    ("quantize", "int8_dot_rows", quantize.int8_dot_rows),        # ref/quantize.py:95
    ("ivf", "probe_centroids", ivf.probe_centroids),              # ref/ivf.py:261
    ("ivf", "search_clusters", ivf.search_clusters),              # ref/ivf.py:285
    ("ivf", "search", ivf.search),                                # ref/ivf.py:337
    ("retrieval", "codesigned_search", retrieval.codesigned_search),  # ref/retrieval.py:110
    ("retrieval", "retrieve", overarch.retrieve),                 # ref/retrieval.py:163
    ("serve", "_reduce_topk", serve._reduce_topk),                # ref/serve.py:98
]


def _filtra_modules():
    pkg = importlib.import_module("filtra")
    for info in pkgutil.iter_modules(pkg.__path__):
        importlib.import_module(f"filtra.{info.name}")
    return [m for name, m in sorted(sys.modules.items())
            if m is not None and (name == "filtra" or name.startswith("filtra."))]


def install(only=None) -> list[tuple[object, str, object]]:
    """Patch the reference. ``only``: optional set of function names to patch. Returns the
    record for ``uninstall`` (module, attribute, original)."""
    mods = _filtra_modules()
    record = []
    for mod_name, fn_name, new in PATCHES:
        if only is not None and fn_name not in only:
            continue
        orig = getattr(importlib.import_module(f"filtra.{mod_name}"), fn_name)
        if orig is new:
            continue
        for m in mods:
            for attr, val in list(vars(m).items()):
                if val is orig:
                    setattr(m, attr, new)
                    record.append((m, attr, orig))
    return record


def uninstall(record) -> None:
    for m, attr, orig in reversed(record):
        setattr(m, attr, orig)
