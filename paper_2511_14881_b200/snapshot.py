"""``FLTRSNP1`` snapshot -> device layout.

Reads the reference's single-file serving artifact (ref/snapshot.py:32-55 format; sections
4-8 = quantized items, quantisation parameters, Bloom planes, validity, item ids; 1-3 =
centroids, permutation, cluster offsets; 9 = embedding cache; 10-12 = scorer, value model,
vocabulary) and materialises it straight into the device structures of this package: a
``DeviceIndex`` (items padded to whole 256-slot tiles and 32-byte rows, planes, validity,
ids, centroids, cluster offsets), a ``DeviceCache`` and a ``DeviceScorer``. The header and
every section checksum (blake2b-64) are verified exactly as the reference loader does
(ref/snapshot.py:192-289), raising the reference's error types.
"""

from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import dataclass
from pathlib import Path
from types import SimpleNamespace

import numpy as np

from .bloom import BloomIndex, BloomParams
from .engine import DeviceIndex
from .errors import BadMagic, ChecksumMismatch, TruncatedSnapshot, VersionUnsupported
from .overarch import DeviceCache, DeviceScorer
from .quantize import QuantParams

MAGIC = b"FLTRSNP1"
FORMAT_VERSION = 1
(SEC_CENTROIDS, SEC_PERM, SEC_CLUSTER_OFFSETS, SEC_ITEMS_Q, SEC_QUANT_PARAMS, SEC_BLOOM_PLANES,
 SEC_VALID_MASK, SEC_ITEM_IDS, SEC_EMBEDDING_CACHE, SEC_SCORER, SEC_VALUE_MODEL,
 SEC_VOCAB) = range(1, 13)
_HEADER_FMT = "<8sIQIQQIIII"  # magic, fmt, snap_ver, dim, n_items, n_slots, k, M, K, scheme
_HEADER_SIZE = struct.calcsize(_HEADER_FMT)
_ENTRY_FMT = "<IQQQ"          # section id, offset, length, checksum
_ENTRY_SIZE = struct.calcsize(_ENTRY_FMT)


def _checksum(data) -> int:
    return int.from_bytes(hashlib.blake2b(data, digest_size=8).digest(), "little")


def describe(path) -> dict:
    """Header and section table (reference ``snapshot.describe``)."""
    info, _ = _header(memoryview(Path(path).read_bytes()))
    return info


def _header(blob: memoryview):
    if len(blob) < _HEADER_SIZE + 4:
        raise TruncatedSnapshot("file shorter than header")
    magic, fmt, ver, dim, n_items, n_slots, k, m, kh, scheme = struct.unpack_from(
        _HEADER_FMT, blob, 0)
    if magic != MAGIC:
        raise BadMagic(f"bad magic {bytes(magic)!r}")
    if fmt != FORMAT_VERSION:
        raise VersionUnsupported(fmt)
    (n_sec,) = struct.unpack_from("<I", blob, _HEADER_SIZE)
    end = _HEADER_SIZE + 4 + n_sec * _ENTRY_SIZE
    if len(blob) < end:
        raise TruncatedSnapshot("file ends inside the section table")
    sections = [struct.unpack_from(_ENTRY_FMT, blob, _HEADER_SIZE + 4 + i * _ENTRY_SIZE)
                for i in range(n_sec)]
    info = {"format_version": fmt, "snapshot_version": ver, "dim": dim, "n_items": n_items,
            "n_slots": n_slots, "n_clusters": k, "bloom_m": m, "bloom_k": kh,
            "hash_scheme_id": scheme,
            "sections": [{"id": s, "offset": o, "length": n, "checksum": c}
                         for s, o, n, c in sections]}
    return info, end


def read_host(path) -> dict:
    """Verified host view of a snapshot: header info and numpy arrays / JSON specs."""
    blob = memoryview(bytearray(Path(path).read_bytes()))  # writable: arrays view it
    info, _ = _header(blob)
    sec = {}
    for e in info["sections"]:
        off, n = e["offset"], e["length"]
        if off + n > len(blob):
            raise TruncatedSnapshot(f"section {e['id']} extends past end of file")
        data = blob[off:off + n]
        if _checksum(data) != e["checksum"]:
            raise ChecksumMismatch(e["id"])
        sec[e["id"]] = data

    def arr(sid, dtype, shape):
        try:
            a = np.frombuffer(sec[sid], dtype=dtype)
        except KeyError as exc:
            raise TruncatedSnapshot(f"missing section {sid}") from exc
        if a.size != int(np.prod(shape)):
            raise TruncatedSnapshot(f"section {sid} has {a.size} elements, expected "
                                    f"{int(np.prod(shape))}")
        return a.reshape(shape)

    n, d, c, words = info["n_slots"], info["dim"], info["n_clusters"], (info["n_slots"] + 63) // 64
    out = {"info": info,
           "centroids": arr(SEC_CENTROIDS, "<f4", (c, d)),
           "perm": arr(SEC_PERM, "<i8", (n,)),
           "cluster_offsets": arr(SEC_CLUSTER_OFFSETS, "<u8", (c, 2)),
           "items_q": arr(SEC_ITEMS_Q, "i1", (n, d)),
           "planes": arr(SEC_BLOOM_PLANES, "<u8", (info["bloom_m"], words)),
           "valid": arr(SEC_VALID_MASK, "<u8", (words,)),
           "item_ids": arr(SEC_ITEM_IDS, "<u8", (n,))}
    try:
        out["qp"] = struct.unpack("<dd", sec[SEC_QUANT_PARAMS])
        cb = sec[SEC_EMBEDDING_CACHE]
        cdim, ncache = struct.unpack_from("<IQ", cb, 0)
        o = struct.calcsize("<IQ")
        out["cache_ids"] = np.frombuffer(cb[o:o + 8 * ncache], dtype="<u8")
        out["cache_vectors"] = np.frombuffer(cb[o + 8 * ncache:], dtype="<f4").reshape(ncache, cdim)
        out["scorer"] = json.loads(bytes(sec[SEC_SCORER]).decode("utf-8"))
        out["value_model"] = json.loads(bytes(sec[SEC_VALUE_MODEL]).decode("utf-8"))
        out["vocab"] = json.loads(bytes(sec[SEC_VOCAB]).decode("utf-8"))
    except KeyError as exc:
        raise TruncatedSnapshot(f"missing section {exc}") from exc
    except (struct.error, ValueError) as exc:
        raise TruncatedSnapshot(str(exc)) from exc
    return out


def scorer_from_spec(spec: dict):
    """Reference-shaped scorer object from the snapshot's scorer JSON
    (ref/scoring.py:163-203), for ``DeviceScorer.from_reference``."""
    f32 = lambda a: np.asarray(a, dtype=np.float32)  # noqa: E731
    if spec.get("kind") == "mlp":
        heads = {n: SimpleNamespace(weight=f32(h["w"]), bias=float(h["b"]))
                 for n, h in spec.get("heads", {}).items()}
        sh = spec.get("shared_head")
        return SimpleNamespace(hidden=tuple((f32(l["w"]), f32(l["b"])) for l in spec.get("hidden", [])),
                               heads=heads,
                               shared_head=SimpleNamespace(weight=f32(sh["w"]), bias=float(sh["b"]))
                               if sh else None)
    if spec.get("kind") == "mol":
        return SimpleNamespace(components=tuple((f32(c["u"]), f32(c["i"])) for c in spec["components"]),
                               gate_weight=f32(spec["gate"]["w"]), gate_bias=f32(spec["gate"]["b"]))
    raise ValueError(f"unknown scorer kind {spec.get('kind')!r}")


@dataclass
class DeviceSnapshot:
    info: dict
    index: DeviceIndex
    cache: DeviceCache
    scorer: DeviceScorer
    value_model: dict | None
    vocab: dict
    perm: np.ndarray


def load_device(path) -> DeviceSnapshot:
    """Verify a snapshot and materialise it in HBM, ready for ``TopkOp`` / ``IvfSearchOp`` /
    ``MultiTaskOp``."""
    h = read_host(path)
    info = h["info"]
    params = BloomParams(m_bits=info["bloom_m"], k_hashes=info["bloom_k"],
                         hash_scheme_id=info["hash_scheme_id"])
    bloom = BloomIndex(params, np.ascontiguousarray(h["planes"]), info["n_slots"])
    index = DeviceIndex.from_arrays(
        np.ascontiguousarray(h["items_q"]), np.ascontiguousarray(h["valid"]),
        np.ascontiguousarray(h["item_ids"]), bloom=bloom, qp=QuantParams(*h["qp"]),
        cluster_offsets=np.asarray(h["cluster_offsets"], dtype=np.int64),
        centroids=np.ascontiguousarray(h["centroids"]))
    cache = DeviceCache(np.ascontiguousarray(h["cache_ids"]), np.ascontiguousarray(h["cache_vectors"]))
    scorer = DeviceScorer.from_reference(scorer_from_spec(h["scorer"]))
    return DeviceSnapshot(info=info, index=index, cache=cache, scorer=scorer,
                          value_model=h["value_model"], vocab=h["vocab"], perm=h["perm"].copy())


__all__ = ["describe", "read_host", "load_device", "DeviceSnapshot", "scorer_from_spec"]
