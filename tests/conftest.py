"""Shared fixtures.  ``-m gpu`` tests need a B200 (run through gpurun);
everything else runs on the CPU build container.

The independent oracles used by the tests live in ``oracle/`` (a CPU
restatement of the reference, pinned to golden vectors the reference
produced: tests/golden/make_golden.py)."""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:
    sys.path.insert(0, str(TESTS))

SEED = int(os.environ.get("MESHLOOP_SEED", "0"))
GOLDEN = TESTS / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run under gpurun)")


@pytest.fixture
def rng():
    return np.random.default_rng(SEED)


class Golden:
    """Lazy access to one golden npz file plus its JSON index."""

    def __init__(self, name: str):
        self.z = np.load(GOLDEN / name)
        self.index = json.loads(bytes(self.z["__index__"]))

    def __getitem__(self, key):
        return self.z[key]

    def __contains__(self, key):
        return key in self.z.files

    def keys(self, prefix: str):
        return [k for k in self.z.files if k.startswith(prefix)]


_golden_cache: dict = {}


def golden(name: str) -> Golden:
    if name not in _golden_cache:
        _golden_cache[name] = Golden(name)
    return _golden_cache[name]


def golden_bytes() -> dict:
    return json.loads((GOLDEN / "bytes.json").read_text())


def import_reference():
    """The stock reference package ``meshloop``: the driver's install under
    ``baseline/_ref`` (travels to the GPU box), else the read-only source tree
    of this container; None if neither is present.  Imported under its own
    name, so ``meshloop.apps`` kernels keep their reference qualified names."""
    import importlib
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "meshloop" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            mod = importlib.import_module("meshloop")
            importlib.import_module("meshloop.apps")
            return mod
    return None


@pytest.fixture(scope="session")
def R():
    mod = import_reference()
    if mod is None:
        pytest.skip("stock reference package not available (baseline/_ref)")
    return mod
