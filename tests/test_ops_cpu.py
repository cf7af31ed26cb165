"""The custom-op boundary and the reference drop-in without a GPU: fake-tensor shapes of
``torch.ops.filtra_b200.*``, the reference-type binding, and the integration installer."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch
from torch._subclasses.fake_tensor import FakeTensorMode

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def test_ops_registered_with_fake_kernels():
    from paper_2511_14881_b200 import ops  # noqa: F401
    for name in ("filtered_topk", "merge_topk", "quantize"):
        assert hasattr(torch.ops.filtra_b200, name)
    with FakeTensorMode():
        q = torch.empty((8, 128), dtype=torch.int8, device="cuda")
        ids, sc, cnt = torch.ops.filtra_b200.filtered_topk(1, q, 100, [], [], [], 0)
        assert (ids.shape, ids.dtype, sc.dtype, cnt.shape) == ((8, 100), torch.int64,
                                                               torch.int32, (8,))
        x = torch.empty((8, 100), dtype=torch.float32, device="cuda")
        assert torch.ops.filtra_b200.quantize(x, -1.0, 1.0, 128).shape == (8, 128)
        s = torch.empty((4, 8, 50), dtype=torch.int32, device="cuda")
        i = torch.empty((4, 8, 50), dtype=torch.int64, device="cuda")
        c = torch.empty((4, 8), dtype=torch.int32, device="cuda")
        out = torch.ops.filtra_b200.merge_topk(s, i, c, 70)
        assert [tuple(t.shape) for t in out] == [(8, 70), (8, 70), (8,)]


def test_filter_meta_round_trip():
    import numpy as np
    from paper_2511_14881_b200 import BloomParams, FilterBatch, compile_filter, workload
    rng = np.random.default_rng(7)
    cfs = [compile_filter(workload.four_attribute_filter(rng), BloomParams()) for _ in range(4)]
    fb = FilterBatch.pack(cfs, BloomParams())
    meta = fb.meta()
    assert len(meta) == len(FilterBatch.META_FIELDS)
    assert meta[0] == 4 and meta[8] == 1  # four queries, CNF form
    with pytest.raises(ValueError):
        FilterBatch.struct_from([torch.zeros(1)], meta)


def _run(code: str, **env) -> str:
    e = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF), str(ROOT)]), **env)
    return subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                          check=True, cwd=ROOT).stdout


@pytest.mark.skipif(not (REF / "filtra").is_dir(), reason="baseline/_ref not installed")
def test_reference_types_bound_when_importable():
    out = _run("import filtra, paper_2511_14881_b200 as fb;"
               "print(fb.TopkResult is filtra.ivf.TopkResult,"
               " fb.errors.DimMismatch is filtra.errors.DimMismatch,"
               " fb.ScanStats is filtra.ivf.ScanStats, fb.FilterStats is filtra.bloom.FilterStats)")
    assert out.split() == ["True"] * 4
    out = _run("import filtra, paper_2511_14881_b200 as fb;"
               "print(fb.TopkResult is filtra.ivf.TopkResult)", FB_REFERENCE_TYPES="0")
    assert out.split() == ["False"]


@pytest.mark.skipif(not (REF / "filtra").is_dir(), reason="baseline/_ref not installed")
def test_integration_install_patches_every_binding():
    out = _run(
        "import filtra, filtra.ivf, filtra.retrieval, filtra.serve\n"
        "from paper_2511_14881_b200 import integration, ivf, retrieval, serve\n"
        "orig = filtra.ivf.search_clusters\n"
        "rec = integration.install()\n"
        "assert filtra.ivf.search_clusters is ivf.search_clusters\n"
        "assert filtra.retrieval.search_clusters is ivf.search_clusters\n"
        "assert filtra.retrieval.codesigned_search is retrieval.codesigned_search\n"
        "assert filtra.serve._reduce_topk is serve._reduce_topk\n"
        "names = {f for _, f, _ in integration.PATCHES}\n"
        "patched = {a for _, a, _ in rec}\n"
        "assert names <= patched, names - patched\n"
        "integration.uninstall(rec)\n"
        "assert filtra.ivf.search_clusters is orig\n"
        "print('ok', len(rec))\n")
    assert out.startswith("ok")


def test_identity_cache_unhashable_dataclass():
    """Reference engine parts are eq-dataclasses (unhashable): the device-copy caches key
    them by identity and drop the entry when the host object is collected."""
    import gc
    from dataclasses import dataclass

    import numpy as np

    from paper_2511_14881_b200._device import IdentityCache

    @dataclass
    class Part:
        data: np.ndarray

    c = IdentityCache()
    a, b = Part(np.zeros(3)), Part(np.zeros(3))
    made = []
    assert c.get_or_make(a, lambda o: made.append(1) or "A") == "A"
    assert c.get_or_make(a, lambda o: made.append(1) or "A2") == "A"
    assert c.get_or_make(b, lambda o: made.append(1) or "B") == "B"
    assert len(made) == 2
    del a
    gc.collect()
    assert len(c._d) == 1
    # objects without weakref support are held strongly, LRU-bounded
    s = IdentityCache(max_strong=2)
    objs = [(i,) for i in range(3)]
    for o in objs:
        s.put(o, o[0])
    assert s.get(objs[0]) is None and s.get(objs[2]) == 2


def test_value_model_code_postfix():
    """The value-model compiler (fb_value_model's bytecode) folds n-ary ops left to right as
    the reference evaluates them (ref value_model.py:75-124) and rejects unknown tasks."""
    import pytest

    from paper_2511_14881_b200.errors import UnknownTask
    from paper_2511_14881_b200.overarch import mean_of_tasks_spec, value_model_code
    code, consts = value_model_code(mean_of_tasks_spec(["a", "b", "c"]), ["a", "b", "c"])
    # CONST(1/3) TASK a TASK b ADD TASK c ADD MUL
    assert code == [0, 1, 1 | (1 << 8), 2, 1 | (2 << 8), 2, 4] and consts == [1 / 3]
    spec = {"op": "if", "cond": {"left": {"op": "task", "task": "b"}, "cmp": ">=",
                                 "right": {"op": "const", "value": 2.0}},
            "then": {"op": "clamp", "args": [{"op": "task", "task": "a"}], "lo": -1, "hi": 1},
            "else": {"op": "div", "args": [{"op": "task", "task": "a"},
                                           {"op": "task", "task": "b"}]}}
    code, consts = value_model_code(spec, ["a", "b"])
    assert code == [1 | (1 << 8), 0, 1, 8 | (1 << 8), 1, 1 | (1 << 8), 5, 12]
    assert consts == [2.0, -1.0, 1.0]
    with pytest.raises(UnknownTask):
        value_model_code({"op": "task", "task": "z"}, ["a"])
    deep = {"op": "task", "task": "a"}
    for _ in range(20):  # right-nested: the stack grows by one per level
        deep = {"op": "add", "args": [{"op": "task", "task": "a"}, deep]}
    assert value_model_code(deep, ["a"]) is None  # deeper than the kernel's stack
