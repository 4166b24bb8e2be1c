"""PTMX matrices and OfflineBundle directories (io.hpp:23-75,
bundle.cpp:49-141) — host I/O of the device path."""
import json
import os

import numpy as np
import pytest

from paper_2103_01983_b200 import bundle
from paper_2103_01983_b200.api import ConfigError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ptmx_v1_3x2.ptmx")


def test_golden_ptmx_reads_column_major_with_time_fields():
    mf = bundle.read_matrix(GOLDEN)
    np.testing.assert_array_equal(mf.data, 0.5 * np.array([[1.0, 4.0], [2.0, 5.0], [3.0, 6.0]]))
    assert mf.dt == 1e-3 and mf.t0 == 0.25


def test_write_reproduces_golden_bytes(tmp_path):
    p = tmp_path / "m.ptmx"
    bundle.write_matrix(p, 0.5 * np.array([[1.0, 4.0], [2.0, 5.0], [3.0, 6.0]]), 1e-3, 0.25)
    assert p.read_bytes() == open(GOLDEN, "rb").read()


def test_roundtrip_and_vectors(tmp_path):
    rng = np.random.default_rng(0)
    m = rng.standard_normal((17, 5))
    bundle.write_matrix(tmp_path / "a.ptmx", m)
    np.testing.assert_array_equal(bundle.read_matrix(tmp_path / "a.ptmx").data, m)
    v = rng.standard_normal(9)
    bundle.write_matrix(tmp_path / "v.ptmx", v)
    np.testing.assert_array_equal(bundle.read_vector(tmp_path / "v.ptmx"), v)
    with pytest.raises(ConfigError, match="expected a single column"):
        bundle.read_vector(tmp_path / "a.ptmx")


def test_read_errors(tmp_path):
    with pytest.raises(ConfigError, match="cannot open"):
        bundle.read_matrix(tmp_path / "missing.ptmx")
    raw = open(GOLDEN, "rb").read()
    (tmp_path / "magic.ptmx").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ConfigError, match="is not a matrix file"):
        bundle.read_matrix(tmp_path / "magic.ptmx")
    (tmp_path / "ver.ptmx").write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(ConfigError, match="unsupported version 2"):
        bundle.read_matrix(tmp_path / "ver.ptmx")
    (tmp_path / "trunc.ptmx").write_bytes(raw[:-8])
    with pytest.raises(ConfigError, match="truncated file"):
        bundle.read_matrix(tmp_path / "trunc.ptmx")


def synthetic_bundle(rng, n=40, m=3, mr=4, nc=5, u=6, nt=4):
    mem = [sorted(rng.choice(n, size=3, replace=False).tolist()) for _ in range(nc)]
    mem_off, mem_ids = bundle._csr(mem)
    cl_off, cl_list = bundle._csr([[0, 2], [1], [], [3, 4, 0]])
    d_off, d_list = bundle._csr([[0], [1, 2], [5], [3, 4]])
    return bundle.OfflineBundle(
        config={"n": n, "modes": m, "name": "synthetic"}, basis_phi=rng.standard_normal((2 * n, m)),
        basis_sv=np.arange(m, 0, -1.0), basis_xref=rng.standard_normal(2 * n),
        residual_phi=rng.standard_normal((2 * n, mr)), residual_sv=np.ones(mr), gnat_a=rng.standard_normal((mr, 2 * nt)),
        sample_ids=np.array([1, 5, 9, 30]), phi_tilde=rng.standard_normal((2 * nc, m)),
        x0_tilde=rng.standard_normal(2 * nc), gamma_tilde=rng.standard_normal(nc),
        cluster_node_ids=np.arange(nc, dtype=np.int32) * 3, mem_off=mem_off, mem_ids=mem_ids,
        zero_gamma=np.array([0, 1, 0, 0, 0], np.uint8), target_ids=np.array([1, 5, 9, 30]), cl_off=cl_off,
        cl_list=cl_list, d_off=d_off, d_list=d_list, direct_ids=np.array([0, 2, 3, 7, 8, 11]),
        direct_phi=rng.standard_normal((2 * u, m)), direct_x0=rng.standard_normal(2 * u),
        direct_gamma=rng.standard_normal(u), training_hashes=[2**63 + 5], training_runs=[{"mu": 1.0}],
        stats={"build_seconds": 0.5})


def test_bundle_save_load_roundtrip(tmp_path):
    b = synthetic_bundle(np.random.default_rng(1))
    b.save(tmp_path / "bundle")
    idx = json.load(open(tmp_path / "bundle" / "index.json"))
    assert list(idx)[:5] == ["format", "version", "config", "matrices", "sample_ids"]
    assert idx["clusters"]["membership"][0] == [int(v) for v in b.mem_ids[:3]]
    assert idx["targets"]["clusters"][2] == []
    c = bundle.OfflineBundle.load(tmp_path / "bundle")
    for k in ("basis_phi", "basis_sv", "basis_xref", "residual_phi", "gnat_a", "sample_ids", "phi_tilde",
              "x0_tilde", "gamma_tilde", "cluster_node_ids", "mem_off", "mem_ids", "zero_gamma", "target_ids",
              "cl_off", "cl_list", "d_off", "d_list", "direct_ids", "direct_phi", "direct_x0", "direct_gamma"):
        np.testing.assert_array_equal(getattr(c, k), getattr(b, k), err_msg=k)
    assert c.config == b.config and c.training_hashes == b.training_hashes and c.stats == b.stats


def test_bundle_load_errors(tmp_path):
    with pytest.raises(ConfigError, match="cannot open"):
        bundle.OfflineBundle.load(tmp_path)
    (tmp_path / "index.json").write_text('{"format": "other"}')
    with pytest.raises(ConfigError, match="not a bundle directory"):
        bundle.OfflineBundle.load(tmp_path)
