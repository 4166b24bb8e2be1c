"""Barnes–Hut quadtree on the B200 vs the oracle (quadtree.hpp:15-308).

Topology (bounds, width, children, begin/end, depth, perm, slot, leaf_node)
and cluster lists must be byte-equal; centroids / Γ sums are bit-equal for
nodes up to the sequential-sum threshold and within 1e-13 above it;
velocities and Jacobians within 1e-12 relative (north_star)."""
import os

import numpy as np
import pytest

from paper_2103_01983_b200 import workloads

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
TOPO = ("bounds", "width", "children", "begin", "end", "depth", "perm", "slot", "leaf_node")


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def random_points(rng, n, scale=10.0, dups=True):
    px = rng.uniform(-scale, scale, n)
    py = rng.uniform(-scale, scale, n)
    if dups and n >= 7:  # test_quadtree.cpp:194-195 duplicates
        px[3] = px[4] = px[1]
        py[3] = py[4] = py[1]
    return px, py


def assert_same_tree(gt, ot, seq_max=2048):
    """Topology byte-equal; Γ sums / centroids bit-equal on nodes with at most
    seq_max members (sequential sums), within 1e-13 on larger nodes."""
    e = gt.export()
    assert gt.num_nodes == ot.num_nodes
    for k in TOPO:
        np.testing.assert_array_equal(e[k], getattr(ot, k), err_msg=k)
    np.testing.assert_array_equal(e["fallback"], ot.fallback)
    small = (ot.end - ot.begin) <= seq_max
    np.testing.assert_array_equal(e["gamma_sum"][small], ot.gamma_sum[small])
    np.testing.assert_array_equal(e["centroid"][small], ot.centroid[small])
    big = ~small
    if big.any():
        assert np.max(np.abs(e["gamma_sum"][big] - ot.gamma_sum[big]) / (np.abs(ot.gamma_sum[big]) + 1e-300)) <= 1e-13
        assert np.max(np.abs(e["centroid"][big] - ot.centroid[big])) <= 1e-13 * (1 + np.max(np.abs(ot.centroid)))


@pytest.mark.parametrize("n", [1, 2, 7, 40, 150, 1000, 5000])
@pytest.mark.parametrize("cap", [1, 4, 16, 32])
def test_random_tree_topology_byte_equal(pt, oracle, n, cap):
    from paper_2103_01983_b200.tree import QuadTree
    rng = np.random.default_rng(11 * n + cap)
    px, py = random_points(rng, n)
    g = rng.uniform(0.1, 2.0, n)
    assert_same_tree(QuadTree(px, py, g, cap), oracle.Tree(px, py, g, cap))


def test_known_answer_four_corners(pt, oracle):
    # test_quadtree.cpp:133-155: preorder ids 1..4 for SW, SE, NW, NE
    from paper_2103_01983_b200.tree import QuadTree
    t = QuadTree([0, 1, 0, 1], [0, 0, 1, 1], np.ones(4), 1)
    assert t.num_nodes == 5
    np.testing.assert_array_equal(t.children[0], [1, 2, 3, 4])
    assert list(t.slot) == [0, 1, 2, 3]


def test_known_answer_split_line_goes_lower_left(pt, oracle):
    # test_quadtree.cpp:157-172
    from paper_2103_01983_b200.tree import QuadTree
    t = QuadTree([0, 2, 1], [0, 2, 1], np.ones(3), 1)
    c = t.children[0]
    assert c[0] >= 0 and c[1] == -1 and c[2] == -1 and c[3] >= 0
    assert t.end[c[0]] - t.begin[c[0]] == 2
    assert_same_tree(t, oracle.Tree([0, 2, 1], [0, 2, 1], np.ones(3), 1))


def test_known_answer_depth_guard_and_degenerate_hull(pt, oracle):
    # test_quadtree.cpp:174-186: coincident points stop at depth 64, root width 1
    from paper_2103_01983_b200.tree import QuadTree
    t = QuadTree([4.5] * 3, [-2.0] * 3, np.ones(3), 1)
    assert t.width[0] == 1.0
    assert t.depth.max() == 64
    leaf = t.leaf_node[0]
    assert t.end[leaf] - t.begin[leaf] == 3
    assert_same_tree(t, oracle.Tree([4.5] * 3, [-2.0] * 3, np.ones(3), 1))


def test_known_answer_zero_net_circulation_fallback(pt):
    # test_quadtree.cpp:204-215
    from paper_2103_01983_b200.tree import QuadTree
    t = QuadTree([0, 1], [0, 1], [1.0, -1.0], 2)
    assert t.fallback[0] == 1 and t.gamma_sum[0] == 0.0
    np.testing.assert_allclose(t.centroid[0], [0.5, 0.5])


def test_build_validation(pt):
    from paper_2103_01983_b200.tree import QuadTree
    with pytest.raises(pt.ConfigError):
        QuadTree([0.0, 1.0], [0.0, 1.0], [1.0, 1.0], 0)
    with pytest.raises(pt.ConfigError):
        QuadTree([0.0, np.nan], [0.0, 1.0], [1.0, 1.0], 1)


CRITERIA = [(0, 0.7), (0, 0.5), (0, 0.0), (1, 1.0), (1, 0.0)]


@pytest.mark.parametrize("kind,value", CRITERIA)
def test_collect_clusters_byte_equal(pt, oracle, kind, value):
    # test_quadtree.cpp:257-287 shape, compared list-for-list with the oracle
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    rng = np.random.default_rng(29)
    n = 3000
    px, py = random_points(rng, n)
    g = rng.uniform(0.1, 2.0, n)
    gt, ot = QuadTree(px, py, g, 4), oracle.Tree(px, py, g, 4)
    crit = ClusterCriterion(kind, value)
    targets = np.r_[0:50, n - 50:n, rng.integers(0, n, 100)]
    co, cl, do, di = gt.collect_clusters_many(targets, crit)
    for j, t in enumerate(targets):
        on, od = ot.collect_clusters(int(t), kind, value)
        np.testing.assert_array_equal(cl[co[j]:co[j + 1]], on)
        np.testing.assert_array_equal(di[do[j]:do[j + 1]], od)


@pytest.mark.parametrize("kind,value", CRITERIA)
@pytest.mark.parametrize("form", [0, 1])
def test_bh_velocity_and_jacobian_parity(pt, oracle, kind, value, form):
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    rng = np.random.default_rng(47)
    n = 4000
    px, py = random_points(rng, n, dups=False)
    g = rng.uniform(0.1, 2.0, n)
    x = np.r_[px, py]
    inflow = rng.uniform(-1, 1, 2 * n)
    sys_ = pt.ParticleSystem(g, 0.05, inflow, form)
    gt, ot = QuadTree(px, py, g, 8), oracle.Tree(px, py, g, 8)
    crit = ClusterCriterion(kind, value)
    f = gt.bh_velocity(x, sys_, crit)
    ref = ot.bh_velocity(x, g, 0.05, kind, value, form, inflow, threads=THREADS)
    assert rel(f, ref) <= 1e-12
    j = gt.bh_jacobian(x, pt.ParticleSystem(g, 0.05, None, form), crit)
    rj = ot.bh_jacobian(x, g, 0.05, kind, value, form)
    assert rel(np.stack([j.dfx_dx, j.dfx_dy, j.dfy_dx, j.dfy_dy]), rj) <= 1e-12


def test_theta_zero_matches_pairwise(pt):
    # test_quadtree.cpp:289-315
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    rng = np.random.default_rng(47)
    n = 200
    px, py = random_points(rng, n, dups=False)
    s = pt.ParticleSystem(rng.uniform(0.1, 2.0, n), 0.05)
    x = np.r_[px, py]
    naive = pt.pairwise_velocity(x, s)
    t = QuadTree(px, py, s.circulation, 4)
    assert np.max(np.abs(t.bh_velocity(x, s, ClusterCriterion.barnes_hut(0.0)) - naive)) <= 1e-12
    assert np.max(np.abs(t.bh_velocity(x, s, ClusterCriterion.neighbor(1e9)) - naive)) <= 1e-12
    flat = QuadTree(px, py, s.circulation, n)
    assert np.max(np.abs(flat.bh_velocity(x, s, ClusterCriterion.barnes_hut(0.0)) - naive)) <= 1e-12


def test_pair_counter_matches_reference(pt, oracle):
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    rng = np.random.default_rng(3)
    n = 500
    px, py = random_points(rng, n, dups=False)
    g = rng.uniform(0.1, 2.0, n)
    t = QuadTree(px, py, g, 4)
    ot = oracle.Tree(px, py, g, 4)
    expect = sum(sum(len(a) for a in ot.collect_clusters(i, 0, 0.5)) for i in range(n))
    pt.reset_kernel_eval_count()
    t.bh_velocity(np.r_[px, py], pt.ParticleSystem(g, 0.05), ClusterCriterion.barnes_hut(0.5))
    assert pt.kernel_eval_count() == expect


def test_config3_two_patches_full_size(pt, oracle):
    """BASELINE configs[2] at full N = 1,048,576, leaf 32, θ = 0.5: byte-equal
    topology, cluster lists on 400 targets, velocities on 2,000 target rows."""
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    w = workloads.config3()
    n = w.n
    px, py = w.x0[:n], w.x0[n:]
    gt, ot = QuadTree(px, py, w.gamma, 32), oracle.Tree(px, py, w.gamma, 32)
    if "PTROM_TREE_BUILD" not in os.environ:  # the measured path: no silent fall back to the level build
        assert build_info(gt.ctx)[0] == 1
    assert_same_tree(gt, ot)
    crit = ClusterCriterion.barnes_hut(0.5)
    rng = np.random.default_rng(3)
    targets = rng.integers(0, n, 400)
    co, cl, do, di = gt.collect_clusters_many(targets, crit)
    for j, t in enumerate(targets):
        on, od = ot.collect_clusters(int(t), 0, 0.5)
        np.testing.assert_array_equal(cl[co[j]:co[j + 1]], on)
        np.testing.assert_array_equal(di[do[j]:do[j + 1]], od)
    f = gt.bh_velocity(w.x0, pt.ParticleSystem(w.gamma, w.delta), crit)
    for b in (0, n // 2 - 1000):
        ref = ot.bh_velocity(w.x0, w.gamma, w.delta, 0, 0.5, t_begin=b, t_end=b + 1000, threads=THREADS)
        rows = np.r_[b:b + 1000, n + b:n + b + 1000]
        assert rel(f[rows], ref[rows]) <= 1e-12


def test_inexact_nodes_certified_and_resolved(pt, oracle):
    """Force block-reduced (inexact) sums on every node above 4 members and pick
    θ equal to an exact opening ratio of the reference: the borderline test
    must be detected, resolved with the exact sequential sums, and the lists
    must still equal the reference's byte for byte."""
    import paper_2103_01983_b200 as ptm
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    rng = np.random.default_rng(5)
    n = 2000
    px, py = random_points(rng, n, dups=False)
    g = rng.uniform(0.1, 2.0, n)
    ot = oracle.Tree(px, py, g, 2)
    # an exactly attainable ratio width/dist for (target 17, some large node)
    tx, ty = px[17], py[17]
    big = [i for i in range(ot.num_nodes) if ot.end[i] - ot.begin[i] > 40 and not (ot.begin[i] <= ot.slot[17] < ot.end[i])]
    node = big[len(big) // 2]
    dx, dy = ot.centroid[node, 0] - tx, ot.centroid[node, 1] - ty
    theta = float(ot.width[node] / np.sqrt(dx * dx + dy * dy))
    os.environ["PTROM_TREE_SEQ_MAX"] = "4"
    try:
        ctx = ptm.Context(0)
    finally:
        del os.environ["PTROM_TREE_SEQ_MAX"]
    gt = QuadTree(px, py, g, 2, ctx=ctx)
    crit = ClusterCriterion.barnes_hut(theta)
    targets = np.arange(0, n, 7)
    targets = np.r_[17, targets]
    co, cl, do, di = gt.collect_clusters_many(targets, crit)
    for j, t in enumerate(targets):
        on, od = ot.collect_clusters(int(t), 0, theta)
        np.testing.assert_array_equal(cl[co[j]:co[j + 1]], on)
        np.testing.assert_array_equal(di[do[j]:do[j + 1]], od)
    assert_same_tree(gt, ot, seq_max=4)


def test_barnes_hut_model_rebuilds(pt, oracle):
    from paper_2103_01983_b200.tree import BarnesHutModel, ClusterCriterion
    w = workloads.config3(n=20000)
    m = BarnesHutModel(pt.ParticleSystem(w.gamma, w.delta), ClusterCriterion.barnes_hut(0.5), 32)
    f = m.velocity(w.x0)
    n = w.n
    ot = oracle.Tree(w.x0[:n], w.x0[n:], w.gamma, 32)
    ref = ot.bh_velocity(w.x0, w.gamma, w.delta, 0, 0.5, threads=THREADS)
    assert rel(f, ref) <= 1e-12


def test_wide_counter_path_above_2pow21(pt, oracle):
    """n + 1 >= 2^21 takes the uint4 quadrant counters (below, three 21-bit
    counters packed in a u64): topology still byte-equal, velocities 1e-12."""
    from paper_2103_01983_b200.tree import ClusterCriterion, QuadTree
    n = (1 << 21) + 5
    rng = np.random.default_rng(21)
    px, py = rng.normal(0, 0.3, n), rng.normal(0, 0.3, n)
    g = rng.uniform(0.1, 1.0, n) / n
    gt, ot = QuadTree(px, py, g, 32), oracle.Tree(px, py, g, 32)
    assert_same_tree(gt, ot)
    x = np.concatenate([px, py])
    f = gt.bh_velocity(x, pt.ParticleSystem(g, 1e-6), ClusterCriterion.barnes_hut(0.5))
    ref = ot.bh_velocity(x, g, 1e-6, 0, 0.5, t_begin=0, t_end=1500, threads=THREADS)
    rows = np.r_[0:1500, n:n + 1500]
    assert rel(f[rows], ref[rows]) <= 1e-12


@pytest.mark.parametrize("n,shards", [(5000, 3), (65536, 8)])
def test_sharded_barnes_hut_slots_equal_full_evaluation(pt, oracle, n, shards):
    """Replicated build + slot-range far field (ShardedBarnesHut's per-rank call,
    SURVEY.md §8e): the slot shards, scattered through perm, are bit-identical
    to the single-call evaluation, and perm is the oracle's."""
    import ctypes as C

    import torch

    from paper_2103_01983_b200.sharded import CudaBhBackend, ShardedBarnesHut, shard_bounds
    w = workloads.config3(n=n)
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    ctx = pt.default_context()
    full = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    cnt = C.c_uint64()
    ctx.check(ctx.lib.ptrom_dev_barnes_hut_velocity_f64(ctx.handle, n, x.data_ptr(), g.data_ptr(), w.delta, 0, 0,
                                                        0.5, 32, None, full.data_ptr(), C.byref(cnt)))
    be = CudaBhBackend()
    fx, fy = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
    perm = None
    for r in range(shards):
        lo, hi = shard_bounds(n, r, shards)
        loc, perm = be.slots(x, g, w.delta, 0, 0, 0.5, 32, None, lo, hi)
        fx[lo:hi], fy[lo:hi] = loc[:hi - lo], loc[hi - lo:]
    f = torch.empty_like(full)
    f[perm.long()] = fx
    f[n + perm.long()] = fy
    np.testing.assert_array_equal(f.cpu().numpy(), full.cpu().numpy())
    f1 = ShardedBarnesHut(n, be).velocity(x, g, w.delta, 0, 0.5, 32)
    np.testing.assert_array_equal(f1.cpu().numpy(), full.cpu().numpy())
    if n <= 5000:
        ot = oracle.Tree(w.x0[:n], w.x0[n:], w.gamma, 32)
        np.testing.assert_array_equal(perm.cpu().numpy(), ot.perm)
        assert rel(full.cpu().numpy(), ot.bh_velocity(w.x0, w.gamma, w.delta, 0, 0.5)) <= 1e-12


def build_info(ctx):
    import ctypes
    m, lv = ctypes.c_int(), ctypes.c_int()
    ctx.check(ctx.lib.ptrom_tree_build_info(ctx.handle, ctypes.byref(m), ctypes.byref(lv)))
    return m.value, lv.value


@pytest.mark.parametrize("case", ["config3", "uniform", "clustered", "cap4_distinct", "seq64"])
def test_morton_build_equals_level_build(pt, case):
    """The Morton-key build and the level-by-level build produce the same
    tree bit for bit (every exported array, sums included), and the Morton
    path is the one taken for these inputs."""
    import paper_2103_01983_b200 as ptm
    from paper_2103_01983_b200.tree import QuadTree
    rng = np.random.default_rng(7)
    cap = 32
    if case == "config3":
        w = workloads.config3(n=200_000)
        px, py, g = w.x0[:w.n], w.x0[w.n:], w.gamma
    elif case == "uniform":
        n = 100_003
        px, py, g = rng.uniform(-3, 5, n), rng.uniform(-1, 1, n), rng.normal(0, 1, n)
    elif case == "clustered":
        n = 150_000
        c = rng.integers(0, 6, n)
        px = rng.normal(0, 0.02, n) + c * 0.3
        py = rng.normal(0, 0.02, n) - c * 0.1
        g = rng.uniform(-1, 1, n)
    elif case == "cap4_distinct":
        n, cap = 20_000, 4
        px, py, g = rng.uniform(0, 1, n), rng.uniform(0, 1, n), rng.uniform(0.5, 1.5, n)
    else:  # small exact-sum threshold: many large (certified) levels
        n, cap = 50_000, 8
        px, py, g = rng.normal(0, 1, n), rng.normal(0, 1, n), rng.uniform(0.5, 1.5, n)
    seq = "64" if case == "seq64" else None
    forced = os.environ.pop("PTROM_TREE_BUILD", None)  # this test picks the build itself
    if seq:
        os.environ["PTROM_TREE_SEQ_MAX"] = seq
    try:
        ctx_m = ptm.Context(0)
    finally:
        os.environ.pop("PTROM_TREE_SEQ_MAX", None)
        if forced is not None:
            os.environ["PTROM_TREE_BUILD"] = forced
    tm = QuadTree(px, py, g, cap, ctx=ctx_m)
    morton, levels = build_info(ctx_m)
    assert morton == 1 and levels > 1
    os.environ["PTROM_TREE_BUILD"] = "levels"
    if seq:
        os.environ["PTROM_TREE_SEQ_MAX"] = seq
    try:
        ctx_l = ptm.Context(0)
    finally:
        os.environ.pop("PTROM_TREE_BUILD", None)
        os.environ.pop("PTROM_TREE_SEQ_MAX", None)
        if forced is not None:
            os.environ["PTROM_TREE_BUILD"] = forced
    tl = QuadTree(px, py, g, cap, ctx=ctx_l)
    assert build_info(ctx_l)[0] == 0
    em, el = tm.export(), tl.export()
    assert tm.num_nodes == tl.num_nodes
    assert set(em) == set(el)
    # nodes above seq_max take certified block sums whose order follows each
    # build's member layout: equal within the certified bound, not bitwise
    small = (el["end"] - el["begin"]) <= int(seq or 2048)
    for k in em:
        if k in ("gamma_sum", "centroid"):
            np.testing.assert_array_equal(em[k][small], el[k][small], err_msg=k)
            np.testing.assert_allclose(em[k][~small], el[k][~small], rtol=1e-12, atol=1e-15, err_msg=k)
        else:
            np.testing.assert_array_equal(em[k], el[k], err_msg=k)


def test_morton_build_falls_back_on_deep_trees(pt, oracle):
    """Coincident points with leaf_capacity 1 need the depth-64 guard, deeper
    than the 32 key levels: the level build takes over, same tree."""
    from paper_2103_01983_b200.tree import QuadTree
    rng = np.random.default_rng(3)
    n = 300
    px, py = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    px[10:14] = px[9]
    py[10:14] = py[9]
    g = rng.uniform(0.5, 1.5, n)
    gt = QuadTree(px, py, g, 1)
    assert build_info(gt.ctx)[0] == 0
    assert_same_tree(gt, oracle.Tree(px, py, g, 1))


def test_morton_build_deterministic_and_small_sizes(pt, oracle):
    """Two Morton builds of the same input are identical array for array, and
    sizes around the subtree / leaf thresholds (1, 33, 2047..2049, 4097)
    still equal the reference."""
    from paper_2103_01983_b200.tree import QuadTree
    rng = np.random.default_rng(99)
    for n in (1, 33, 2047, 2048, 2049, 4097):
        px, py = rng.normal(0, 1, n), rng.normal(0, 1, n)
        g = rng.uniform(0.5, 1.5, n)
        a, b = QuadTree(px, py, g, 32), QuadTree(px, py, g, 32)
        ea, eb = a.export(), b.export()
        for k in ea:
            np.testing.assert_array_equal(ea[k], eb[k], err_msg=f"{k} n={n}")
        assert_same_tree(a, oracle.Tree(px, py, g, 32))
