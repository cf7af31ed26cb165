"""FLTRSNP1 snapshot loader: host verification against the reference's own file (header,
checksums, error types) on CPU, and the device materialisation on the GPU driving the
config-5 multi-task path to the reference's retrieve() output."""

from __future__ import annotations

import shutil

import numpy as np
import pytest

from conftest import GOLDEN, json_to_expr, load_json


def test_snapshot_describe_matches_reference():
    from paper_2511_14881_b200 import snapshot
    ref = load_json("snapshot_small.json")["describe"]
    assert snapshot.describe(GOLDEN / "snapshot_small.fsnap") == ref
    h = snapshot.read_host(GOLDEN / "snapshot_small.fsnap")
    assert h["items_q"].shape == (ref["n_slots"], ref["dim"])
    assert h["planes"].shape == (ref["bloom_m"], (ref["n_slots"] + 63) // 64)
    assert h["scorer"]["kind"] == "mol" and h["value_model"]["op"] == "add"


def test_snapshot_corruption_raises_reference_errors(tmp_path):
    from paper_2511_14881_b200 import snapshot
    from paper_2511_14881_b200.errors import BadMagic, ChecksumMismatch, TruncatedSnapshot
    src = GOLDEN / "snapshot_small.fsnap"
    blob = bytearray(src.read_bytes())
    bad = tmp_path / "bad.fsnap"
    flipped = bytearray(blob)
    flipped[-100] ^= 0xFF
    bad.write_bytes(bytes(flipped))
    with pytest.raises(ChecksumMismatch):
        snapshot.read_host(bad)
    magic = bytearray(blob)
    magic[0:8] = b"NOTASNAP"
    bad.write_bytes(bytes(magic))
    with pytest.raises(BadMagic):
        snapshot.read_host(bad)
    bad.write_bytes(bytes(blob[: len(blob) // 2]))
    with pytest.raises(TruncatedSnapshot):
        snapshot.read_host(bad)
    shutil.copy(src, tmp_path / "ok.fsnap")
    snapshot.read_host(tmp_path / "ok.fsnap")


@pytest.mark.gpu
def test_snapshot_to_device_multitask_matches_reference(cuda):
    import torch
    import paper_2511_14881_b200 as fb
    from paper_2511_14881_b200 import snapshot
    snap = snapshot.load_device(GOLDEN / "snapshot_small.fsnap")
    assert snap.scorer.kind == "dot"  # the published default: identity mixture of logits
    fx = load_json("snapshot_small.json")
    for r in fx["requests"]:
        op = fb.MultiTaskOp(snap.index, snap.cache, 1, ["a", "b"], 200, 50,
                            scorer=snap.scorer, value_model=snap.value_model)
        cf = fb.compile_filter(json_to_expr(r["expr"]), fb.BloomParams())
        users = torch.as_tensor(np.array(r["users"], dtype=np.float32)[None], device="cuda")
        out = op(users, op.pack_filters([cf]).to_device())
        torch.cuda.synchronize()
        ids, scores, _ = out.host(0)
        assert ids.tolist() == r["ids"]
        assert [float(x).hex() for x in scores] == r["scores"]
