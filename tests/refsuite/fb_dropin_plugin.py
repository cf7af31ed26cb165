"""pytest plugin for running the REFERENCE's own test suite against the B200 drop-in:
patches the reference's hot-path functions (paper_2511_14881_b200.integration.install)
before any test module is collected, so the tests' ``from filtra.ivf import ...`` bind the
GPU implementations. Used by tests/test_reference_suite.py in a subprocess."""

from __future__ import annotations

_RECORD = []


def pytest_configure(config):
    import os
    os.environ.setdefault("FB_GRAPH_STRICT", "1")
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the drop-in needs a CUDA device")
    from paper_2511_14881_b200 import integration
    _RECORD.extend(integration.install())
    patched = sorted({f"{m.__name__}.{a}" for m, a, _ in _RECORD})
    config._fb_patched = patched
    # also on stdout: ``-q`` runs (tests/test_reference_suite.py) suppress report headers
    print("B200 drop-in patched: " + ", ".join(patched), flush=True)


def pytest_report_header(config):
    return ["B200 drop-in patched: " + ", ".join(getattr(config, "_fb_patched", []))]
