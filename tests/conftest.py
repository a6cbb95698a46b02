import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_PARITY = []


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built libmci.so")


@pytest.fixture
def parity_log():
    """record(name, rel_errors, **extra): per-row relative L2 errors of a full-size parity
    subset; written with max / median to $MCI_PARITY_LOG (JSON) at the end of the session."""
    def record(name, rel, **extra):
        import numpy as np
        rel = np.asarray(rel, dtype=np.float64).ravel()
        _PARITY.append(dict(name=name, n=int(rel.size), max=float(rel.max()), median=float(np.median(rel)),
                            **extra))
    return record


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("MCI_PARITY_LOG")
    if path and _PARITY:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as fh:
            json.dump(_PARITY, fh, indent=1)
