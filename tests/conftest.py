import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    # a fresh on-disk cache (compiled cubins, chosen pass groupings) per test
    # session, so every run exercises the planner and NVRTC as built
    if "HISVSIM_CACHE_DIR" not in os.environ:
        import tempfile

        os.environ["HISVSIM_CACHE_DIR"] = tempfile.mkdtemp(prefix="hisvsim_test_cache_")


class Golden:
    """Lazy access to the committed reference fixtures (tests/golden)."""

    def __init__(self):
        self._cache = {}

    def json(self, name):
        if name not in self._cache:
            self._cache[name] = json.loads((GOLDEN / f"{name}.json").read_text())
        return self._cache[name]

    def npz(self, name):
        key = name + ".npz"
        if key not in self._cache:
            self._cache[key] = dict(np.load(GOLDEN / f"{name}.npz"))
        return self._cache[key]


@pytest.fixture(scope="session")
def golden():
    return Golden()


def parts_of(doc):
    return [(tuple(g), tuple(q)) for g, q in doc]


def partition_of(doc, strategy="golden", limit=0):
    from paper_2205_06973_b200.partition import Part, PartitionResult

    return PartitionResult(strategy, limit, tuple(Part(i, tuple(g), tuple(q)) for i, (g, q) in enumerate(doc)))
