"""Shared fixtures.  `gpu` tests need a B200 (sm_100a) and run via gpurun;
everything else runs on the CPU-only build container."""

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100a device (run with -m gpu on the B200 box)")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    opener = gzip.open if name.endswith(".gz") else open
    with opener(path, "rt") as f:
        return json.load(f)


SCHED_FAMILIES = [
    "sched_known.json",
    "sched_random500.json.gz",
    "sched_baseline.json.gz",
    "sched_warm100.json.gz",
    "sched_base.json.gz",
    "sched_asym.json.gz",
]


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture
def ring4_placement():
    from paper_2511_16947_b200 import Placement

    return Placement(4, ((0, 3), (0, 1), (1, 2), (2, 3)), (0, 0, 1, 1))


@pytest.fixture
def ring4_loads():
    from paper_2511_16947_b200 import LoadMatrix

    return LoadMatrix(((4, 0, 0, 0), (0, 6, 0, 0), (0, 0, 14, 0), (0, 0, 0, 8)))


@pytest.fixture
def identical4_placement():
    from paper_2511_16947_b200 import Placement

    return Placement(4, ((0, 2), (0, 2), (1, 3), (1, 3)), (0, 1, 0, 1))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture
def tune():
    """tune(ffn_pair=1, ...) sets library launch-tuning fields (hep_tuning_set) for
    the test; the previous values are restored afterwards."""
    from paper_2511_16947_b200 import _lib

    saved = _lib.get_tuning()
    yield lambda **kw: _lib.set_tuning(**kw)
    _lib.set_tuning(**saved)
