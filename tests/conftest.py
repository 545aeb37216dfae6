import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large configs (c3..c5 builds)")


@pytest.fixture(scope="session")
def ico3():
    import paper_2605_00429_b200 as P
    V, F = P.icosphere(3)
    return V, F, P.HostEngine.build(V, F)


@pytest.fixture(scope="session")
def c1():
    import paper_2605_00429_b200 as P
    V, F = P.mesh_config(1)
    return V, F, P.HostEngine.build(V, F)


@pytest.fixture(scope="session")
def c2():
    import paper_2605_00429_b200 as P
    V, F = P.mesh_config(2)
    return V, F, P.HostEngine.build(V, F)
