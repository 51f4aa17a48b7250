import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: multi-second CPU oracle cases")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def eng():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2203_02507_b200 as fpm
    return fpm.default_engine(0)
