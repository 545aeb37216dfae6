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


def oracle_checker(arrays):
    """The CPU checker of the GPU tests: the reference's own point-triangle kernel (oracle/_ref:
    REF/proj/src/geom.cpp compiled where it lies + the restated query loop) when it was built, else
    the C restatement (pinned bit-for-bit to it by tests/test_oracle_pin.py)."""
    import oracle as O
    return O.OracleEngine(arrays, reference=O.have_reference())


_big = {}


def big_config(cfg):
    """c3..c5 engines, built once per session (each build takes minutes)."""
    if cfg not in _big:
        import paper_2605_00429_b200 as P
        V, F = P.mesh_config(cfg)
        _big[cfg] = (V, F, P.HostEngine.build(V, F))
    return _big[cfg]
