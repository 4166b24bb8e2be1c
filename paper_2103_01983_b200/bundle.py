"""Reference-format PTMX matrices and OfflineBundle directories (SURVEY.md §8f
row 4), so the device path consumes what the reference's offline stage writes
and emits trajectories the reference's tools read.

    read_matrix / write_matrix      io.hpp:23-75   (PTMX v1)
    OfflineBundle.load / save       bundle.cpp:49-141, bundle.hpp:15-27
    OfflineBundle.to_device()       → PODBasis, GnatOperator, SurrogateSourceBasis
    OfflineBundle.from_device(...)  ← the device offline producers

PTMX layout (little-endian, io.hpp:23-51): 4-byte magic "PTMX", u32 version
(1), u64 rows, u64 cols, f64 dt, f64 t0, then rows*cols f64 column-major.
This is host I/O around the device path; nothing here computes.
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from .api import ConfigError

MAGIC = b"PTMX"
VERSION = 1
_HEADER = struct.Struct("<4sIQQdd")  # 40 bytes


@dataclass
class MatrixFile:  # io.hpp:29-33
    data: np.ndarray  # (rows, cols), Fortran order
    dt: float = 0.0
    t0: float = 0.0


def write_matrix(path, mat, dt: float = 0.0, t0: float = 0.0) -> None:
    """io.hpp:35-51. 1-D input is written as a single column (bundle.cpp:11-13)."""
    a = np.asarray(mat, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.ndim != 2:
        raise ConfigError("write_matrix: expected a matrix")
    try:
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, VERSION, a.shape[0], a.shape[1], float(dt), float(t0)))
            f.write(np.asfortranarray(a).tobytes(order="F"))
    except OSError:
        raise ConfigError(f"write_matrix: cannot open {path}") from None


def read_matrix(path) -> MatrixFile:
    """io.hpp:53-75 with the reference's error messages."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise ConfigError(f"read_matrix: cannot open {path}") from None
    if len(raw) < _HEADER.size:
        raise ConfigError(f"read_matrix: {path} is not a matrix file")
    magic, version, rows, cols, dt, t0 = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ConfigError(f"read_matrix: {path} is not a matrix file")
    if version != VERSION:
        raise ConfigError(f"read_matrix: unsupported version {version}")
    need = rows * cols * 8
    if len(raw) - _HEADER.size < need:
        raise ConfigError(f"read_matrix: truncated file {path}")
    data = np.frombuffer(raw, dtype="<f8", count=rows * cols, offset=_HEADER.size)
    return MatrixFile(data.reshape((rows, cols), order="F").copy(order="F"), float(dt), float(t0))


def read_vector(path) -> np.ndarray:  # bundle.cpp:15-19
    m = read_matrix(path).data
    if m.shape[1] != 1:
        raise ConfigError(f"{path}: expected a single column")
    return m[:, 0].copy()


def _csr(lists) -> tuple[np.ndarray, np.ndarray]:
    off = np.zeros(len(lists) + 1, np.int64)
    for k, l in enumerate(lists):
        off[k + 1] = off[k] + len(l)
    flat = np.fromiter((int(v) for l in lists for v in l), dtype=np.int64, count=int(off[-1]))
    return off, flat


def _nested(off, flat) -> list:
    return [[int(v) for v in flat[off[k]:off[k + 1]]] for k in range(len(off) - 1)]


_MATRICES = ["basis_phi.ptmx", "basis_sv.ptmx", "basis_xref.ptmx", "residual_phi.ptmx", "residual_sv.ptmx",
             "gnat_a.ptmx", "surrogate_phi.ptmx", "surrogate_x0.ptmx", "surrogate_gamma.ptmx", "direct_phi.ptmx",
             "direct_x0.ptmx", "direct_gamma.ptmx"]


@dataclass
class OfflineBundle:  # bundle.hpp:15-27
    config: Any  # ExperimentConfig JSON (kept verbatim; the control plane is out of scope)
    basis_phi: np.ndarray
    basis_sv: np.ndarray
    basis_xref: np.ndarray
    residual_phi: np.ndarray
    residual_sv: np.ndarray
    gnat_a: np.ndarray
    sample_ids: np.ndarray
    phi_tilde: np.ndarray
    x0_tilde: np.ndarray
    gamma_tilde: np.ndarray
    cluster_node_ids: np.ndarray
    mem_off: np.ndarray
    mem_ids: np.ndarray
    zero_gamma: np.ndarray
    target_ids: np.ndarray
    cl_off: np.ndarray
    cl_list: np.ndarray
    d_off: np.ndarray
    d_list: np.ndarray
    direct_ids: np.ndarray
    direct_phi: np.ndarray
    direct_x0: np.ndarray
    direct_gamma: np.ndarray
    training_hashes: list = field(default_factory=list)
    training_runs: Any = field(default_factory=list)
    stats: Any = None

    # -------------------------------------------------------------- I/O ---
    def save(self, directory) -> None:
        """bundle.cpp:49-94: twelve PTMX files + index.json (same keys and order)."""
        os.makedirs(directory, exist_ok=True)
        mats = [self.basis_phi, self.basis_sv, self.basis_xref, self.residual_phi, self.residual_sv, self.gnat_a,
                self.phi_tilde, self.x0_tilde, self.gamma_tilde, self.direct_phi, self.direct_x0, self.direct_gamma]
        for name, m in zip(_MATRICES, mats):
            write_matrix(os.path.join(directory, name), m)
        index = {
            "format": "ptrom-bundle",
            "version": 1,
            "config": self.config,
            "matrices": list(_MATRICES),
            "sample_ids": [int(v) for v in self.sample_ids],
            "clusters": {
                "node_ids": [int(v) for v in self.cluster_node_ids],
                "membership": _nested(self.mem_off, self.mem_ids),
                "zero_gamma": [int(v != 0) for v in self.zero_gamma],
            },
            "targets": {
                "ids": [int(v) for v in self.target_ids],
                "clusters": _nested(self.cl_off, self.cl_list),
                "direct": _nested(self.d_off, self.d_list),
            },
            "direct_ids": [int(v) for v in self.direct_ids],
            "training_hashes": [int(v) for v in self.training_hashes],
            "training_runs": self.training_runs,
            "stats": self.stats,
        }
        try:
            with open(os.path.join(directory, "index.json"), "w") as f:
                json.dump(index, f, indent=2)
                f.write("\n")
        except OSError:
            raise ConfigError(f"save_json: cannot open {os.path.join(directory, 'index.json')}") from None

    @staticmethod
    def load(directory) -> "OfflineBundle":
        """bundle.cpp:96-141."""
        path = os.path.join(directory, "index.json")
        try:
            with open(path) as f:
                index = json.load(f)
        except OSError:
            raise ConfigError(f"load_json: cannot open {path}") from None
        except ValueError as e:
            raise ConfigError(f"load_json: {path}: {e}") from None
        if not isinstance(index, dict) or index.get("format", "") != "ptrom-bundle":
            raise ConfigError(f"{directory}: not a bundle directory")
        j = lambda name: os.path.join(directory, name)
        try:
            cl, tg = index["clusters"], index["targets"]
            mem_off, mem_ids = _csr(cl["membership"])
            cl_off, cl_list = _csr(tg["clusters"])
            d_off, d_list = _csr(tg["direct"])
            b = OfflineBundle(
                config=index["config"],
                basis_phi=read_matrix(j("basis_phi.ptmx")).data,
                basis_sv=read_vector(j("basis_sv.ptmx")),
                basis_xref=read_vector(j("basis_xref.ptmx")),
                residual_phi=read_matrix(j("residual_phi.ptmx")).data,
                residual_sv=read_vector(j("residual_sv.ptmx")),
                gnat_a=read_matrix(j("gnat_a.ptmx")).data,
                sample_ids=np.asarray(index["sample_ids"], np.int64),
                phi_tilde=read_matrix(j("surrogate_phi.ptmx")).data,
                x0_tilde=read_vector(j("surrogate_x0.ptmx")),
                gamma_tilde=read_vector(j("surrogate_gamma.ptmx")),
                cluster_node_ids=np.asarray(cl["node_ids"], np.int32),
                mem_off=mem_off, mem_ids=mem_ids,
                zero_gamma=np.asarray([int(z) != 0 for z in cl["zero_gamma"]], np.uint8),
                target_ids=np.asarray(tg["ids"], np.int64),
                cl_off=cl_off, cl_list=cl_list, d_off=d_off, d_list=d_list,
                direct_ids=np.asarray(index["direct_ids"], np.int64),
                direct_phi=read_matrix(j("direct_phi.ptmx")).data,
                direct_x0=read_vector(j("direct_x0.ptmx")),
                direct_gamma=read_vector(j("direct_gamma.ptmx")),
            )
        except KeyError as e:
            raise ConfigError(f"{directory}: bundle index is missing {e}") from None
        b.training_hashes = [int(h) for h in index.get("training_hashes", [])]
        b.training_runs = index.get("training_runs", [])
        b.stats = index.get("stats")
        b.validate()
        return b

    def validate(self) -> None:
        nd, m = self.basis_phi.shape
        if nd % 2:
            raise ConfigError("bundle: state dimension must be even")
        if self.basis_xref.shape[0] != nd or self.basis_sv.shape[0] != m:
            raise ConfigError("bundle: basis shape mismatch")
        nc = self.gamma_tilde.shape[0]
        if self.phi_tilde.shape[0] != 2 * nc or self.x0_tilde.shape[0] != 2 * nc:
            raise ConfigError("bundle: surrogate table shape mismatch")
        if len(self.mem_off) != nc + 1 or len(self.zero_gamma) != nc:
            raise ConfigError("bundle: cluster membership count mismatch")
        if len(self.cl_off) != len(self.target_ids) + 1 or len(self.d_off) != len(self.target_ids) + 1:
            raise ConfigError("bundle: per-target list count mismatch")
        if self.gnat_a.shape[1] != 2 * len(self.sample_ids):
            raise ConfigError("bundle: GNAT operator does not match the sample count")

    # ----------------------------------------------------------- device ---
    def to_device(self, ctx=None):
        """→ (PODBasis, GnatOperator, SurrogateSourceBasis) resident on the B200
        (the GnatSolver / hyperpair inputs, rom.hpp:264-290)."""
        from .rom import GnatOperator, PODBasis, SurrogateSourceBasis
        basis = PODBasis(self.basis_phi, self.basis_sv, self.basis_xref, ctx=ctx)
        op = GnatOperator(basis, self.sample_ids, self.gnat_a)
        sur = SurrogateSourceBasis.from_tables(
            self.phi_tilde, self.gamma_tilde, self.x0_tilde, self.zero_gamma, self.mem_off, self.mem_ids,
            self.target_ids, self.cl_off, self.cl_list, self.direct_ids, self.direct_phi, self.direct_x0,
            self.direct_gamma, self.d_off, self.d_list, ctx=basis.ctx)
        return basis, op, sur

    @staticmethod
    def from_device(config, basis, residual_phi, residual_sv, op, sur, training_hashes=(), training_runs=(),
                    stats=None) -> "OfflineBundle":
        """Packs device-built offline products (greedy_sample, build_gnat_operator,
        cluster_pod) into the reference's bundle layout."""
        lists = sur.export_lists()
        tab = sur.export()
        return OfflineBundle(
            config=config, basis_phi=basis.phi, basis_sv=basis.singular_values, basis_xref=basis.x_ref,
            residual_phi=np.asarray(residual_phi, float), residual_sv=np.asarray(residual_sv, float),
            gnat_a=op.A, sample_ids=op.sample_ids, phi_tilde=tab["phi_tilde"], x0_tilde=tab["x0_tilde"],
            gamma_tilde=tab["gamma_tilde"], cluster_node_ids=lists["cluster_node_ids"], mem_off=lists["mem_off"],
            mem_ids=lists["mem_ids"], zero_gamma=tab["zero_gamma"], target_ids=np.asarray(sur.target_ids, np.int64),
            cl_off=lists["cl_off"], cl_list=lists["cl_list"], d_off=lists["d_off"], d_list=lists["d_list"],
            direct_ids=lists["direct_ids"], direct_phi=lists["direct_phi"], direct_x0=lists["direct_x0"],
            direct_gamma=tab["direct_gamma"], training_hashes=list(training_hashes),
            training_runs=list(training_runs), stats=stats)


def write_trajectory(path, x_hat, dt: float, t0: float = 0.0) -> None:
    """x̂ (M x n_steps) as a time-series PTMX (io.hpp:23-26: dt/t0 set)."""
    write_matrix(path, x_hat, dt, t0)


# ------------------------------------------------------------------ native --
def _native_lib():
    from . import _lib
    return _lib.load()


def _native_check(rc, ctx=None):
    if rc == 0:
        return
    msg = (ctx.lib.ptrom_last_error(ctx.handle) if ctx is not None else _native_lib().ptrom_io_last_error()).decode()
    if rc == 2:
        raise ConfigError(msg)
    from .api import CudaError, NumericalError
    raise (NumericalError if rc == 3 else CudaError)(msg)


def read_matrix_native(path) -> MatrixFile:
    """io.hpp:53-75 through the C ABI (ptrom_ptmx_read; no GPU needed)."""
    import ctypes as C
    lib = _native_lib()
    rows, cols, dt, t0 = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_double()
    p = os.fsencode(path)
    _native_check(lib.ptrom_ptmx_read(None, p, C.addressof(rows), C.addressof(cols), C.addressof(dt),
                                      C.addressof(t0), None, 0))
    data = np.zeros(max(rows.value * cols.value, 1))
    _native_check(lib.ptrom_ptmx_read(None, p, None, None, None, None, data.ctypes.data, data.shape[0]))
    return MatrixFile(data[:rows.value * cols.value].reshape((rows.value, cols.value), order="F"), dt.value, t0.value)


def write_matrix_native(path, mat, dt: float = 0.0, t0: float = 0.0) -> None:
    """io.hpp:35-51 through the C ABI (ptrom_ptmx_write)."""
    a = np.asarray(mat, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    a = np.asfortranarray(a)
    _native_check(_native_lib().ptrom_ptmx_write(None, os.fsencode(path), a.shape[0], a.shape[1], float(dt),
                                                 float(t0), a.ctypes.data))


def load_native(directory) -> OfflineBundle:
    """bundle.cpp:96-141 through the C ABI (ptrom_bundle_open + _export): the
    loader a C++ host links; returns the same OfflineBundle as load()."""
    import ctypes as C
    lib = _native_lib()
    h = C.c_void_p()
    _native_check(lib.ptrom_bundle_open(None, os.fsencode(directory), C.byref(h)))
    try:
        sz = np.zeros(11, np.int64)
        lib.ptrom_bundle_sizes(h, sz.ctypes.data)
        nd, m, mr, ns, ar, nc, u, nt, nmem, ncl, ndl = (int(v) for v in sz)
        F = lambda r, c: np.zeros((r, c), order="F")
        out = dict(basis_phi=F(nd, m), basis_sv=np.zeros(m), basis_xref=np.zeros(nd), residual_phi=F(nd, mr),
                   residual_sv=np.zeros(mr), gnat_a=F(ar, 2 * ns), sample_ids=np.zeros(ns, np.int64),
                   phi_tilde=F(2 * nc, m), x0_tilde=np.zeros(2 * nc), gamma_tilde=np.zeros(nc),
                   cluster_node_ids=np.zeros(nc, np.int32), mem_off=np.zeros(nc + 1, np.int64),
                   mem_ids=np.zeros(nmem, np.int64), zero_gamma=np.zeros(nc, np.uint8),
                   target_ids=np.zeros(nt, np.int64), cl_off=np.zeros(nt + 1, np.int64),
                   cl_list=np.zeros(ncl, np.int64), d_off=np.zeros(nt + 1, np.int64), d_list=np.zeros(ndl, np.int64),
                   direct_ids=np.zeros(u, np.int64), direct_phi=F(2 * u, m), direct_x0=np.zeros(2 * u),
                   direct_gamma=np.zeros(u))
        order = ["basis_phi", "basis_sv", "basis_xref", "residual_phi", "residual_sv", "gnat_a", "sample_ids",
                 "phi_tilde", "x0_tilde", "gamma_tilde", "cluster_node_ids", "mem_off", "mem_ids", "zero_gamma",
                 "target_ids", "cl_off", "cl_list", "d_off", "d_list", "direct_ids", "direct_phi", "direct_x0",
                 "direct_gamma"]
        _native_check(lib.ptrom_bundle_export(h, *(out[k].ctypes.data if out[k].size else None for k in order)))
        n = lib.ptrom_bundle_config_json(h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib.ptrom_bundle_config_json(h, buf, n + 1)
        config = json.loads(buf.value.decode()) if n > 0 else None
    finally:
        lib.ptrom_bundle_free(h)
    return OfflineBundle(config=config, **out)


def to_device_native(directory, ctx=None):
    """ptrom_bundle_open + ptrom_bundle_to_device: (PODBasis, GnatOperator,
    SurrogateSourceBasis) built by the C loader, no Python table handling."""
    import ctypes as C

    from .api import default_context
    from .rom import GnatOperator, PODBasis, SurrogateSourceBasis
    ctx = ctx or default_context()
    lib = ctx.lib
    h = C.c_void_p()
    _native_check(lib.ptrom_bundle_open(ctx.handle, os.fsencode(directory), C.byref(h)), ctx)
    try:
        sz = np.zeros(11, np.int64)
        lib.ptrom_bundle_sizes(h, sz.ctypes.data)
        nd, m, mr, ns, ar, nc, u, nt = (int(v) for v in sz[:8])
        hb, ho, hs = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _native_check(lib.ptrom_bundle_to_device(ctx.handle, h, C.byref(hb), C.byref(ho), C.byref(hs)), ctx)
        tid = np.zeros(nt, np.int64)
        ids = np.zeros(ns, np.int64)
        lib.ptrom_bundle_export(h, *([None] * 6), ids.ctypes.data, *([None] * 7), tid.ctypes.data, *([None] * 8))
    finally:
        lib.ptrom_bundle_free(h)
    return (PODBasis.adopt(ctx, hb, nd, m), GnatOperator.adopt(ctx, ho, ids),
            SurrogateSourceBasis(ctx, hs, m, nc, u, nt, tid))
