import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built libvest_cuda.so")
    config.addinivalue_line("markers", "slow: longer-running GPU property tests at full BASELINE sizes")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle as O

    if not O.available("port"):
        O.build()
    return O


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, name + ".npz"))


SEQ_CASES = ["seq_543_lf", "seq_543_l1_masked", "seq_876_lf", "seq_2020_10_lf", "seq_4mode_l1",
             "seq_2mode_lf", "seq_5mode_lf", "seq_c1_scaled", "seq_c2_shape"]
