"""The C ABI's PTMX and OfflineBundle I/O (csrc/bundle_io.cu; io.hpp:23-75,
bundle.cpp:96-141) — the loader a C++ host links — against the golden PTMX
bytes and the Python writer. Host code only: runs without a GPU."""
import json
import os

import numpy as np
import pytest

from paper_2103_01983_b200 import bundle
from paper_2103_01983_b200.api import ConfigError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ptmx_v1_3x2.ptmx")


def test_native_reads_golden_ptmx():
    mf = bundle.read_matrix_native(GOLDEN)
    np.testing.assert_array_equal(mf.data, 0.5 * np.array([[1.0, 4.0], [2.0, 5.0], [3.0, 6.0]]))
    assert mf.dt == 1e-3 and mf.t0 == 0.25


def test_native_write_reproduces_golden_bytes(tmp_path):
    p = tmp_path / "m.ptmx"
    bundle.write_matrix_native(p, 0.5 * np.array([[1.0, 4.0], [2.0, 5.0], [3.0, 6.0]]), 1e-3, 0.25)
    assert p.read_bytes() == open(GOLDEN, "rb").read()
    rng = np.random.default_rng(2)
    m = rng.standard_normal((31, 7))
    bundle.write_matrix_native(tmp_path / "a.ptmx", m)
    np.testing.assert_array_equal(bundle.read_matrix(tmp_path / "a.ptmx").data, m)  # Python reader agrees


def test_native_read_errors_use_reference_messages(tmp_path):
    with pytest.raises(ConfigError, match="read_matrix: cannot open"):
        bundle.read_matrix_native(tmp_path / "missing.ptmx")
    raw = open(GOLDEN, "rb").read()
    (tmp_path / "magic.ptmx").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ConfigError, match="is not a matrix file"):
        bundle.read_matrix_native(tmp_path / "magic.ptmx")
    (tmp_path / "ver.ptmx").write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(ConfigError, match="unsupported version 2"):
        bundle.read_matrix_native(tmp_path / "ver.ptmx")
    (tmp_path / "trunc.ptmx").write_bytes(raw[:-8])
    with pytest.raises(ConfigError, match="truncated file"):
        bundle.read_matrix_native(tmp_path / "trunc.ptmx")


def test_native_bundle_load_equals_python_load(tmp_path):
    from test_bundle import synthetic_bundle
    b = synthetic_bundle(np.random.default_rng(1))
    b.save(tmp_path / "bundle")
    c = bundle.load_native(tmp_path / "bundle")
    py = bundle.OfflineBundle.load(tmp_path / "bundle")
    for k in ("basis_phi", "basis_sv", "basis_xref", "residual_phi", "residual_sv", "gnat_a", "sample_ids",
              "phi_tilde", "x0_tilde", "gamma_tilde", "cluster_node_ids", "mem_off", "mem_ids", "zero_gamma",
              "target_ids", "cl_off", "cl_list", "d_off", "d_list", "direct_ids", "direct_phi", "direct_x0",
              "direct_gamma"):
        np.testing.assert_array_equal(getattr(c, k), getattr(py, k), err_msg=k)
    assert c.config == b.config


def test_native_bundle_errors(tmp_path):
    with pytest.raises(ConfigError, match="load_json: cannot open"):
        bundle.load_native(tmp_path)
    (tmp_path / "index.json").write_text('{"format": "other", "config": {}}')
    with pytest.raises(ConfigError, match="not a bundle directory"):
        bundle.load_native(tmp_path)
    from test_bundle import synthetic_bundle
    b = synthetic_bundle(np.random.default_rng(3))
    b.save(tmp_path / "b2")
    idx = json.load(open(tmp_path / "b2" / "index.json"))
    del idx["targets"]["direct"]
    json.dump(idx, open(tmp_path / "b2" / "index.json", "w"))
    with pytest.raises(ConfigError, match="missing"):
        bundle.load_native(tmp_path / "b2")
    b.save(tmp_path / "b3")
    os.remove(tmp_path / "b3" / "gnat_a.ptmx")
    with pytest.raises(ConfigError, match="read_matrix: cannot open"):
        bundle.load_native(tmp_path / "b3")
