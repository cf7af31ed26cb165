"""CPU checks of the k-means host logic (paper_2511_14881_b200.kmeans): the cluster-major slot
layout and the empty-cluster refill, run on CPU tensors against the oracle / the reference's
rules (ref ivf.py:123-130, 229-249)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import filtra_oracle as orc
from paper_2511_14881_b200 import kmeans


def test_ivf_layout_matches_oracle():
    rng = np.random.default_rng(4)
    for n, k in [(1, 1), (63, 2), (64, 1), (65, 3), (1000, 7), (5000, 40)]:
        assign = rng.integers(0, k, size=n)
        if k > 2:
            assign[assign == 1] = 0  # an empty cluster
        ids = rng.integers(0, 2**64, size=n, dtype=np.uint64)
        ids[: n // 3] |= np.uint64(1 << 63)  # ids above 2^63 order as unsigned
        perm, offs = kmeans.ivf_layout(torch.as_tensor(assign), torch.as_tensor(ids.view(np.int64)), k)
        want_perm, want_offs = orc.ivf_layout(assign, ids, k)
        assert np.array_equal(perm.numpy(), want_perm), (n, k)
        assert np.array_equal(offs.numpy().astype(np.uint64), want_offs), (n, k)


def _refill_reference(assign, cost, k):
    """ref ivf.py:123-130 restated: each empty cluster takes the costliest point of the
    first largest cluster."""
    sizes = np.bincount(assign, minlength=k)
    for c in np.flatnonzero(sizes == 0):
        donor = int(np.argmax(sizes))
        members = np.flatnonzero(assign == donor)
        far = members[np.argmax(cost[members])]
        assign[far] = c
        cost[far] = 0.0
        sizes[donor] -= 1
        sizes[c] += 1
    return assign, cost


def test_refill_empty_matches_reference_rule():
    rng = np.random.default_rng(8)
    for n, k in [(10, 4), (50, 9), (300, 30)]:
        assign = rng.integers(0, max(1, k // 3), size=n)      # many empty clusters
        cost = np.round(rng.random(n), 1)                      # ties in the cost
        want_a, want_c = _refill_reference(assign.copy(), cost.copy(), k)
        a, c = torch.as_tensor(assign.copy()), torch.as_tensor(cost.copy())
        kmeans._refill_empty(a, c, k)
        assert np.array_equal(a.numpy(), want_a), (n, k)
        assert np.array_equal(c.numpy(), want_c), (n, k)
