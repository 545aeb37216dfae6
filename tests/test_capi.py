"""The drop-in boundary: every entry point declared in include/p2m.h is exported by the two
in-tree libraries, loads without a GPU, and fails with status codes (never exceptions)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "p2m.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(p2m_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) >= 25
    host, cuda = L.host(), L.cuda()
    missing = []
    for n in names:
        if not (hasattr(host, n) or hasattr(cuda, n)):
            missing.append(n)
    assert not missing, missing


def test_libraries_are_in_tree_and_built_for_sm100a():
    so = os.path.join(ROOT, "paper_2605_00429_b200", "lib", "libp2m_cuda.so")
    assert os.path.exists(so)
    blob = open(so, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


def test_status_codes_not_exceptions():
    host = L.host()
    h = C.c_void_p()
    rc = host.p2m_build(None, 0, None, 0, None, C.byref(h))
    assert rc == -1 and b"null" in host.p2m_last_error()
    cfg = L.BuildConfig()
    host.p2m_build_config_default(C.byref(cfg))
    assert (cfg.augment, cfg.alpha, cfg.k, cfg.rho, cfg.max_rounds, cfg.domain_scale) == (1, 4.0, 24, 0.75, 3, 10.0)
    cfg.k = 0
    V, F = P.icosphere(1)
    rc = host.p2m_build(L.ptr(V), len(V), L.ptr(F.astype(np.uint32), L.u32p), len(F), C.byref(cfg), C.byref(h))
    assert rc == -1
    cuda = L.cuda()
    assert cuda.p2m_query(None, None, 0, None, None, None, None, None, None) == -3  # engine not built
    assert cuda.p2m_engine_info(None, None, None, None) == -3
    n = C.c_int()
    assert cuda.p2m_kernels_per_query(None, 1, C.byref(n)) == -1
    rc = host.p2m_mesh_config(9, C.byref(L.dp()), C.byref(C.c_uint64()), C.byref(L.u32p()), C.byref(C.c_uint64()))
    assert rc == -1


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_engine_create_without_device_fails_loudly():
    V, F = P.icosphere(1)
    h = P.HostEngine.build(V, F)
    with pytest.raises(P.P2MError, match="P2M_ERR_CUDA"):
        P.Engine(h)


def test_engine_desc_invalid():
    d = L.EngineDesc()
    out = C.c_void_p()
    assert L.cuda().p2m_engine_create(C.byref(d), 1, None, C.byref(out)) == -1


def test_header_compiles_as_c_and_cpp(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "p2m.h"\nint main(void){ p2m_counters c; (void)c; return P2M_OK; }\n')
    inc = os.path.join(ROOT, "include")
    assert os.system(f"gcc -std=c99 -Wall -Werror -I{inc} -c {src} -o {tmp_path}/t.o") == 0
    assert os.system(f"g++ -std=c++17 -Wall -Werror -x c++ -I{inc} -c {src} -o {tmp_path}/t2.o") == 0
