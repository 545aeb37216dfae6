"""Host-side logic of bench.py that needs no GPU: the roofline evidence is used only when it was
captured on the same sources and the same row count; the in-line parity counts rows bit by bit."""
import json
import os

import numpy as np

import bench


def test_ncu_evidence_matches_by_source_hash_and_rows(tmp_path, monkeypatch):
    d = tmp_path / "profiles" / "r99" / "final"
    d.mkdir(parents=True)
    ev = {"src_sha256": "abc", "rows": 1000, "dram_bytes_per_launch": 5.0, "issue_slots_pct": 50.0}
    (d / "ncu_scan_c5.json").write_text(json.dumps(ev))
    (d / "ncu_scan_c4.json").write_text("not json")
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    got = bench.ncu_evidence(5, 1000, "abc")
    assert got and got["dram_bytes_per_launch"] == 5.0 and got["file"] == os.path.join("profiles", "r99", "final", "ncu_scan_c5.json")
    assert bench.ncu_evidence(5, 1000, "other build") is None      # another build of the kernels
    assert bench.ncu_evidence(5, 2000, "abc") is None              # another workload size
    assert bench.ncu_evidence(4, 1000, "abc") is None              # unreadable file is skipped
    assert bench.ncu_evidence(3, 1000, "abc") is None              # no capture for this config


def test_source_hash_tracks_the_cuda_sources():
    h = bench.src_sha256()
    assert len(h) == 64 and h == bench.src_sha256()


def test_parity_rows_is_bitwise():
    n = 5
    ref = {"distance": np.arange(n, dtype=np.float64), "closest": np.ones((n, 3)), "face": np.arange(n, dtype=np.uint32),
           "site": np.zeros(n, np.uint32), "flags": np.zeros(n, np.uint32)}
    gpu = {k: v.copy() for k, v in ref.items()}
    assert bench.parity_rows(ref, gpu, n) == n
    gpu["distance"][2] = np.nextafter(gpu["distance"][2], 10.0)   # one ulp off is a mismatch
    gpu["closest"][4, 1] = -1.0
    gpu["face"][0] = 7
    assert bench.parity_rows(ref, gpu, n) == n - 3
    ref["distance"][1] = 0.0
    gpu["distance"][1] = -0.0                                      # signed zero differs in bits
    assert bench.parity_rows(ref, gpu, n) == n - 4
