"""Host mirror of the reference's quadtree interface (quadtree.hpp:15-308,
integrators.hpp:83-102) over the C ABI; the tree lives on the B200.

    ClusterCriterion.barnes_hut(theta) / .neighbor(p_c)   quadtree.hpp:189-203
    QuadTree(px, py, gamma, leaf_capacity)                build_tree, quadtree.hpp:124-162
      .nodes / .perm / .slot / .leaf_node (export)        quadtree.hpp:15-47
      .collect_clusters(target, criterion)                quadtree.hpp:213-252
      .bh_velocity(state, sys, criterion)                 quadtree.hpp:257-281
      .bh_jacobian(state, sys, criterion)                 quadtree.hpp:285-308
    BarnesHutModel(sys, criterion, leaf_capacity)         integrators.hpp:83-102
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .api import BlockDiagonalJacobian, ConfigError, Context, ParticleSystem, _bump, default_context


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


@dataclass(frozen=True)
class ClusterCriterion:  # quadtree.hpp:189-203
    kind: int  # 0 barnes_hut, 1 neighbor
    value: float

    @staticmethod
    def barnes_hut(theta: float) -> "ClusterCriterion":
        if not theta >= 0:
            raise ConfigError("opening ratio must be >= 0")
        return ClusterCriterion(0, float(theta))

    @staticmethod
    def neighbor(p_c: float) -> "ClusterCriterion":
        if not p_c >= 0:
            raise ConfigError("neighborhood width factor must be >= 0")
        return ClusterCriterion(1, float(p_c))


class QuadTree:
    def __init__(self, px, py, gamma, leaf_capacity: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        px, py, g = _f64(px), _f64(py), _f64(gamma)
        if px.shape != py.shape:
            raise ConfigError("build_tree: points must be N x 2")
        if g.shape[0] != px.shape[0]:
            raise ConfigError("build_tree: gamma size mismatch")
        self.n = px.shape[0]
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.ptrom_tree_build_f64(self.ctx.handle, self.n, _p(px), _p(py), _p(g),
                                                         int(leaf_capacity), C.byref(h)))
        self._h = h
        self.num_nodes = int(self.ctx.lib.ptrom_tree_num_nodes(h))
        self._export = None

    def export(self) -> dict:
        if self._export is None:
            nn, n = self.num_nodes, self.n
            e = dict(bounds=np.zeros((nn, 4)), width=np.zeros(nn), centroid=np.zeros((nn, 2)),
                     gamma_sum=np.zeros(nn), children=np.zeros((nn, 4), np.int32), begin=np.zeros(nn, np.int64),
                     end=np.zeros(nn, np.int64), depth=np.zeros(nn, np.int32), fallback=np.zeros(nn, np.uint8),
                     perm=np.zeros(n, np.int64), slot=np.zeros(n, np.int64), leaf_node=np.zeros(n, np.int32))
            self.ctx.check(self.ctx.lib.ptrom_tree_export(
                self.ctx.handle, self._h, *(_p(e[k]) for k in ("bounds", "width", "centroid", "gamma_sum", "children",
                                                               "begin", "end", "depth", "fallback", "perm", "slot",
                                                               "leaf_node"))))
            self._export = e
        return self._export

    def __getattr__(self, name):
        if name in ("bounds", "width", "centroid", "gamma_sum", "children", "begin", "end", "depth", "fallback",
                    "perm", "slot", "leaf_node"):
            return self.export()[name]
        raise AttributeError(name)

    def collect_clusters_many(self, targets, criterion: ClusterCriterion):
        t = np.ascontiguousarray(targets, dtype=np.int64)
        nt = t.shape[0]
        co = np.zeros(nt + 1, np.int64)
        do = np.zeros(nt + 1, np.int64)
        lib, h = self.ctx.lib, self.ctx.handle
        self.ctx.check(lib.ptrom_collect_clusters(h, self._h, criterion.kind, criterion.value, nt, _p(t), _p(co), None,
                                                  0, _p(do), None, 0))
        cl = np.zeros(max(int(co[-1]), 1), np.int32)
        di = np.zeros(max(int(do[-1]), 1), np.int64)
        self.ctx.check(lib.ptrom_collect_clusters(h, self._h, criterion.kind, criterion.value, nt, _p(t), _p(co),
                                                  _p(cl), cl.shape[0], _p(do), _p(di), di.shape[0]))
        return co, cl[:co[-1]], do, di[:do[-1]]

    def collect_clusters(self, target: int, criterion: ClusterCriterion):
        co, cl, do, di = self.collect_clusters_many([target], criterion)
        return cl, di

    def bh_velocity(self, state, sys: ParticleSystem, criterion: ClusterCriterion) -> np.ndarray:
        x, g, inflow = _f64(state), _f64(sys.circulation), _f64(sys.inflow)
        n = g.shape[0]
        if x.shape[0] != 2 * n:
            raise ConfigError(f"bh_velocity: state dimension {x.shape[0]} does not match particle count {n}")
        f = np.empty(2 * n)
        cnt = C.c_uint64()
        self.ctx.check(self.ctx.lib.ptrom_bh_velocity_f64(self.ctx.handle, self._h, n, _p(x), _p(g), float(sys.delta),
                                                          int(sys.kernel_form), criterion.kind, criterion.value,
                                                          _p(inflow), _p(f), C.byref(cnt)))
        _bump(cnt.value)
        return f

    def bh_jacobian(self, state, sys: ParticleSystem, criterion: ClusterCriterion) -> BlockDiagonalJacobian:
        x, g = _f64(state), _f64(sys.circulation)
        n = g.shape[0]
        out = [np.empty(n) for _ in range(4)]
        self.ctx.check(self.ctx.lib.ptrom_bh_jacobian_f64(self.ctx.handle, self._h, n, _p(x), _p(g), float(sys.delta),
                                                          int(sys.kernel_form), criterion.kind, criterion.value,
                                                          *(_p(o) for o in out)))
        return BlockDiagonalJacobian(*out)

    def close(self):
        if getattr(self, "_h", None):
            self.ctx.lib.ptrom_tree_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class BarnesHutModel:  # integrators.hpp:83-102 (tree rebuilt on every call)
    sys: ParticleSystem
    criterion: ClusterCriterion
    leaf_capacity: int

    def velocity(self, x, ctx: Optional[Context] = None) -> np.ndarray:
        ctx = ctx or default_context()
        x, g, inflow = _f64(x), _f64(self.sys.circulation), _f64(self.sys.inflow)
        n = g.shape[0]
        if x.shape[0] != 2 * n:
            raise ConfigError(f"bh_velocity: state dimension {x.shape[0]} does not match particle count {n}")
        f = np.empty(2 * n)
        cnt = C.c_uint64()
        ctx.check(ctx.lib.ptrom_barnes_hut_velocity_f64(ctx.handle, n, _p(x), _p(g), float(self.sys.delta),
                                                        int(self.sys.kernel_form), self.criterion.kind,
                                                        self.criterion.value, int(self.leaf_capacity), _p(inflow),
                                                        _p(f), C.byref(cnt)))
        _bump(cnt.value)
        return f

    def jacobian(self, x):
        n = self.sys.size()
        x = _f64(x)
        return QuadTree(x[:n], x[n:], self.sys.circulation, self.leaf_capacity).bh_jacobian(x, self.sys,
                                                                                           self.criterion)
