import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session")
def tiny():
    import datagen
    return datagen.generate(1, with_sample_queries=50)


@pytest.fixture(scope="session")
def tiny_oracle(tiny):
    from oracle import oracle as O
    c = tiny["cfg"]
    return O.Index(tiny["X"], c.L, c.K, c.N_r, c.index_seed, c.max_size, c.sample_frac)
