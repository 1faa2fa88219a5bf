import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CALIB_PATH = os.path.join(ROOT, "paper_2212_01317_b200", "data", "calib_q0.5.txt")

# a rank that never reaches a collective of libmpr's in-process communicator fails the
# test after 2 minutes instead of the library's 10
os.environ.setdefault("MPR_GROUP_TIMEOUT_S", "120")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmpr.so")
    config.addinivalue_line("markers", "slow: long-running statistical pin")


def read_calibration(path=CALIB_PATH):
    T, e = [], []
    with open(path) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            a, b = line.split()[:2]
            T.append(float.fromhex(a)); e.append(float.fromhex(b))
    return np.array(T, np.float32), np.array(e, np.float32)


@pytest.fixture(scope="session")
def calib():
    return read_calibration()


@pytest.fixture(scope="session")
def toy_table():
    # low-T harmonic line e = -1 + T/4 (SURVEY c.6 worked lattice; tests only)
    return np.array([0.0001, 1.0, 2.0], np.float32), np.array([-0.999975, -0.75, -0.5], np.float32)
