"""bench.py --workload config3 | config4 — the secondary BASELINE.json configs
with the same JSON-line contract as the headline (bench.py, config 2).

config3 (BASELINE configs[2]): one step = BarnesHutModel::velocity
  (integrators.hpp:83-102): tree build + cluster aggregation + far field at
  N = 1,048,576, leaf 32, θ = 0.5, through ptrom_dev_barnes_hut_velocity_f64.
  Metric: bodies/s. Dominant kernel: the far-field traversal (tree_eval.cu),
  FP64 roofline at 12 flops per interaction + 7 per prune test.
config4 (BASELINE configs[3]): one step = a batch of B μ instances marched 50
  steps (5 GN updates each) through ptrom_ptrom_simulate_batch_f64, cycling
  through the 4,096 seeded μ. Metric: instance-steps/s.
  Dominant kernel: hyperpair (rom.cu), 25 flops per interaction.
"""
from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

from bench import ClockSampler, measured_peaks

ROOT = os.path.dirname(os.path.abspath(__file__))
BH_FLOPS_INTERACTION, BH_FLOPS_PRUNE = 12, 7
VJ_FLOPS = 25


def _ncu_traffic(name):
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", name)))
        return float(d["dram_bytes_per_launch"])
    except Exception:
        return None


def _count_launches(fn):
    """Kernels launched by one call of fn (torch profiler / CUPTI), ours only."""
    try:
        import torch
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        # our kernels + the CUB sorts/scans our library launches; not torch's or copies
        ours = [nm for nm in names if "at::" not in nm and "Memset" not in nm and "Memcpy" not in nm
                and "memcpy" not in nm.lower()]
        return len(ours), len(names)
    except Exception:
        return None, None


# Launch counting runs the torch profiler (CUPTI), which stays attached to the
# process afterwards; every count is therefore deferred until all timed
# regions of the run are done (run_deferred_counts).
_DEFERRED = []


def defer_count(line, fn, mult):
    """line["gpu_launches"] = (our kernels launched by one fn()) * mult, later."""
    line["gpu_launches"] = None
    _DEFERRED.append((line, fn, mult))


def run_deferred_counts():
    while _DEFERRED:
        line, fn, mult = _DEFERRED.pop(0)
        ours, _ = _count_launches(fn)
        line["gpu_launches"] = ours * mult if ours is not None else None


def _steps(args, default):
    return args.steps if args.steps_given else default


def run(args, rank, world):
    import torch
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    if world > 1:
        # Barnes-Hut shards the far field by target (one all-gather per
        # evaluation); PTROM splits μ instances (no data-path exchange).
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    if args.workload == "config3":
        line = bench_config3(args, world)
    else:
        line = bench_config4(args, world)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([line["ms_per_step"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["ms_per_step"] = float(t.item())
        # config 3: one N-body evaluation split across ranks (strong scaling);
        # config 4: every rank marches its own μ block (weak scaling)
        strong = line.get("scaling") == "strong"
        line["value"] = line["units_per_step"] * (1 if strong else world) * 1e3 / line["ms_per_step"]
    run_deferred_counts()  # every rank (the sharded step has collectives)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    line.pop("units_per_step", None)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ config 3
def bench_config3(args, world):
    import torch

    import paper_2103_01983_b200 as pt
    from paper_2103_01983_b200 import workloads
    w = workloads.config3()
    n, theta, leaf = w.n, 0.5, 32
    ctx = pt.default_context(torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    f = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cnt = ctypes.c_uint64()

    if world == 1:
        def step():
            ctx.check(lib.ptrom_dev_barnes_hut_velocity_f64(ctx.handle, n, x.data_ptr(), g.data_ptr(), w.delta, 0,
                                                            0, theta, leaf, None, f.data_ptr(), ctypes.byref(cnt)))
    else:
        # replicated build, far field split by tree slot, shards
        # all-gathered over NCCL and scattered back to particle order
        from paper_2103_01983_b200.sharded import CudaBhBackend, ShardedBarnesHut
        sharded = ShardedBarnesHut(n, CudaBhBackend(torch.cuda.current_device()))

        def step():
            f.copy_(sharded.velocity(x, g, w.delta, 0, theta, leaf))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = _steps(args, 20)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    stats = []
    with ClockSampler(torch.cuda.current_device()) as clocks:
        for k in range(K):
            l2_flush.zero_()
            starts[k].record(stream)
            lib.ptrom_profile_begin(ctx.handle)
            step()
            ends[k].record(stream)
            ms, nl = ctypes.c_double(), ctypes.c_int64()
            ctx.check(lib.ptrom_profile_end(ctx.handle, ctypes.byref(ms), ctypes.byref(nl)))
            st = [ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(),
                  ctypes.c_uint64()]
            ctx.check(lib.ptrom_tree_stats(ctx.handle, *(ctypes.byref(v) for v in st)))
            stats.append((ms.value, nl.value, st[0].value, st[1].value, st[2].value, st[3].value, st[4].value))
        torch.cuda.synchronize()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    value = n * K / (total_ms * 1e-3)
    eval_ms = sum(s[0] for s in stats) / max(1, sum(s[1] for s in stats))
    inter, prune = stats[-1][4], stats[-1][5]
    flops = BH_FLOPS_INTERACTION * inter + BH_FLOPS_PRUNE * prune
    achieved = flops / (eval_ms * 1e-3) / 1e12
    peaks = measured_peaks(torch.cuda.current_device())
    build_ms = float(np.median([s[2] for s in stats]))
    nodes = stats[-1][6]
    build_bytes = 36 * n + 136 * nodes  # 24+12 B/body, 112+24 B/node
    hbm = _measured_hbm()
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peaks["fp64_dfma_tflops"] if peaks else None,
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_dfma_tflops"] if peaks else None,
                "traffic": _ncu_traffic("r02_bh_eval_ncu_summary.json"),
                "kernel": "bh_eval_warp_kernel (csrc/tree_eval.cu)", "avg_launch_ms": eval_ms,
                "interactions_per_launch": inter, "prune_tests_per_launch": prune,
                "flops_convention": "12/interaction + 7/prune test (BASELINE.md §2)",
                "peak_source": "measured live: tools/peaks.cu DFMA chain"}
    build_roof = {"bound": "hbm", "median_build_ms": build_ms, "algorithmic_bytes": build_bytes,
                  "achieved_gbs": build_bytes / (build_ms * 1e-3) / 1e9, "peak_gbs": hbm,
                  "frac": (build_bytes / (build_ms * 1e-3) / 1e9) / hbm if hbm else None, "nodes": nodes}
    mi, lv = ctypes.c_int(), ctypes.c_int()
    ctx.check(lib.ptrom_tree_build_info(ctx.handle, ctypes.byref(mi), ctypes.byref(lv)))
    build_roof["build"] = "morton-key sort" if mi.value else "level partition"
    build_roof["note"] = ("latency-bound, not HBM-bound: sequential finish_node chains of the <=2048-member "
                          "nodes, radix passes and level barriers (DESIGN.md section 6)")

    # e2e: host buffers through the drop-in ptrom_barnes_hut_velocity_f64 (one
    # GPU), or pinned host state -> every rank, sharded evaluation, result ->
    # host (N GPUs)
    hx_t = torch.tensor(w.x0).pin_memory()
    hx = hx_t.numpy()
    hg = torch.tensor(w.gamma).pin_memory().numpy()
    hf_t = torch.empty(2 * n, dtype=torch.float64).pin_memory()
    hf = hf_t.numpy()
    if world == 1:
        fn = lambda: ctx.check(lib.ptrom_barnes_hut_velocity_f64(ctx.handle, n, hx.ctypes.data, hg.ctypes.data,
                                                                 w.delta, 0, 0, theta, leaf, None, hf.ctypes.data,
                                                                 ctypes.byref(cnt)))
        api = "ptrom_barnes_hut_velocity_f64 (host buffers)"
    else:
        def fn():
            x.copy_(hx_t, non_blocking=True)
            step()
            hf_t.copy_(f, non_blocking=True)
            torch.cuda.synchronize()
        api = "ShardedBarnesHut.velocity (pinned state in, velocities out on every rank)"
    fn()
    ke = max(3, min(K, 10))
    t0 = time.perf_counter()
    for _ in range(ke):
        fn()
    e2e_s = time.perf_counter() - t0
    e2e = {"value": n * ke / e2e_s, "unit": "bodies/s",
           "h2d_bytes_per_step": int(hx.nbytes + (hg.nbytes if world == 1 else 0)),
           "d2h_bytes_per_step": int(hf.nbytes), "api": api}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_config3(w, theta, leaf, args.cpu_seconds)
    line = {
        "metric": "Barnes-Hut velocity evaluation bodies/s (fp64; build + aggregation + far field)",
        "value": value, "unit": "bodies/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "units_per_step": n, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": w.name, "n": n, "leaf_capacity": leaf, "theta": theta, "delta": w.delta,
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "parallelism": "single GPU" if world == 1 else
                   f"replicated build, far field split by tree slot x{world} (NCCL all-gather)"},
        "e2e": e2e, "roofline": roofline, "build_roofline": build_roof, "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "phase_ms": {"build_median": build_ms, "far_field_avg": eval_ms},
    }
    defer_count(line, step, K)
    return line


def _measured_hbm():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("hbm_gbs", "hbm_burst_gbs", "hbm_sustained_gbs"):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return None


def _cpu_config3(w, theta, leaf, seconds, threads=1):
    """Oracle build_tree on all N bodies + bh_velocity on a bounded target
    sample (1 core, the reference's serial protocol)."""
    from oracle import pyoracle
    n = w.n
    t0 = time.perf_counter()
    tree = pyoracle.Tree(w.x0[:n], w.x0[n:], w.gamma, leaf)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    probe = 2048
    tree.bh_velocity(w.x0, w.gamma, w.delta, 0, theta, t_begin=0, t_end=probe * threads, threads=threads)
    dt = time.perf_counter() - t0
    rows = int(min(n, max(probe * threads, probe * threads * max(1.0, seconds - t_build) / max(dt, 1e-6))))
    t0 = time.perf_counter()
    tree.bh_velocity(w.x0, w.gamma, w.delta, 0, theta, t_begin=0, t_end=rows, threads=threads)
    t_eval = time.perf_counter() - t0
    per_body = t_build / n + t_eval / rows
    return {"value": 1.0 / per_body, "unit": "bodies/s", "cores": threads, "kind": "port",
            "sample": f"oracle build_tree on all {n} bodies ({t_build:.1f} s, 1 thread) + bh_velocity on {rows} "
                      f"targets ({t_eval:.1f} s, {threads} threads); bodies/s = 1 / (build/N + eval/targets)"}


# ------------------------------------------------------------------ config 4
def _config4_setup(args):
    import paper_2103_01983_b200 as pt
    from paper_2103_01983_b200 import rom, workloads
    from paper_2103_01983_b200.tree import ClusterCriterion
    t0 = time.perf_counter()
    w = workloads.config4()
    t_gen = time.perf_counter() - t0
    ctx = pt.default_context()
    t0 = time.perf_counter()
    ids = rom.greedy_sample(w.phi_r, w.n_samples)
    A = rom.build_gnat_operator(w.phi_r, ids)
    g1 = w.gamma_a + w.gamma_b
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, ids, A)
    sur = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
    t_off = time.perf_counter() - t0
    return pt, rom, w, ctx, ids, A, basis, op, sur, {"generate_inputs_host_s": t_gen, "device_offline_s": t_off}


def bench_config4(args, world):
    import torch
    pt, rom, w, ctx, ids, A, basis, op, sur, offline = _config4_setup(args)
    rank = int(os.environ.get("RANK", 0))
    B = args.batch
    n_steps = w.n_steps
    cfg = rom.RomConfig(1e-300, 5, 1.0)  # exactly 5 GN updates, 6 hyperpair calls per step
    grid = pt.TimeGrid(w.dt, n_steps)
    sys_ = pt.ParticleSystem(w.gamma_a + w.gamma_b, w.delta)
    mu_all = np.asarray(w.mu)
    # μ-instance split across ranks (PtromInstanceSplit): rank r takes its block of the 4,096
    lo, hi = rank * len(mu_all) // world, (rank + 1) * len(mu_all) // world
    mu_rank = mu_all[lo:hi]
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    state = {"k": 0}

    def step():
        k = state["k"]
        state["k"] += 1
        sel = np.take(mu_rank, np.arange(k * B, (k + 1) * B), mode="wrap")
        return rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, sel, sys_, grid, cfg, batch=B)

    for _ in range(args.warmup):
        rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, mu_rank[:B], sys_, pt.TimeGrid(w.dt, 1), cfg,
                                 batch=B)
    torch.cuda.synchronize()
    K = _steps(args, max(1, len(mu_rank) // B))
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    pt.reset_kernel_eval_count()
    wall = 0.0
    hp_ms, hp_n = 0.0, 0
    finite = True
    with ClockSampler(torch.cuda.current_device()) as clocks:
        for k in range(K):
            starts[k].record(stream)
            lib.ptrom_profile_begin(ctx.handle)
            t0 = time.perf_counter()
            tr = step()
            wall += time.perf_counter() - t0
            ends[k].record(stream)
            ms, nl = ctypes.c_double(), ctypes.c_int64()
            ctx.check(lib.ptrom_profile_end(ctx.handle, ctypes.byref(ms), ctypes.byref(nl)))
            hp_ms += ms.value
            hp_n += nl.value
            finite = finite and bool(np.all(np.isfinite(tr.x_hat)))
        torch.cuda.synchronize()
    interactions = pt.kernel_eval_count()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    units = B * n_steps
    value = units * K / (total_ms * 1e-3)
    avg_hp_ms = hp_ms / max(1, hp_n)
    inter_per_launch = interactions / max(1, hp_n)
    achieved = VJ_FLOPS * inter_per_launch / (avg_hp_ms * 1e-3) / 1e12
    peaks = measured_peaks(torch.cuda.current_device())
    L = sur.export_lists()
    nt = len(ids)
    srcs = sur.n_clusters + sur.n_direct
    alg_bytes = 16 * B * srcs + 16 * srcs + 4 * (len(L["cl_list"]) + len(L["d_list"])) + 64 * nt * B
    hbm = _measured_hbm()
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peaks["fp64_dfma_tflops"] if peaks else None,
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_dfma_tflops"] if peaks else None,
                "traffic": _ncu_traffic("r02_hyperpair_ncu_summary.json"),
                "kernel": "hyperpair_kernel (csrc/rom.cu)", "avg_launch_ms": avg_hp_ms, "launches": hp_n,
                "interactions_per_launch": inter_per_launch,
                "flops_convention": "25 per fused velocity+Jacobian interaction (BASELINE.md §2)",
                "hbm_view": {"algorithmic_bytes_per_launch": alg_bytes,
                             "achieved_gbs": alg_bytes / (avg_hp_ms * 1e-3) / 1e9, "peak_gbs": hbm},
                # the bound that binds: 16-byte position gathers, one per
                # interaction and lane, against the random-gather rate tools/gather_probe.cu
                # measures for a working set larger than L2 (profiles/r02_gather_probe.txt)
                "gather_view": {"gathered_bytes_per_launch": 16.0 * inter_per_launch,
                                "achieved_tbs": 16.0 * inter_per_launch / (avg_hp_ms * 1e-3) / 1e12,
                                "probe_tbs": 10.83, "frac": 16.0 * inter_per_launch / (avg_hp_ms * 1e-3) / 1e12 / 10.83,
                                "probe": "tools/gather_probe.cu, 537 MB random 512-byte rows"},
                "peak_source": "measured live: tools/peaks.cu DFMA chain"}
    e2e = {"value": units * K / wall, "unit": "instance-steps/s",
           "h2d_bytes_per_step": int(8 * B + 16 * w.n), "d2h_bytes_per_step": int(B * n_steps * (8 * basis.modes() + 5)),
           "api": "ptrom_ptrom_simulate_batch_f64 (host μ, Γa, Γb in; host x̂, iterations, converged out)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_config4(w, ids, A, args.cpu_seconds)
    line = {
        "metric": "PTROM online instance-steps/s (fp64)", "value": value, "unit": "instance-steps/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": total_ms / K, "units_per_step": units,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64; Φ = 16-mode POD of 200 seeded snapshots, SURVEY.md §8d)",
        "config": {"workload": w.name, "n": w.n, "instances_per_step": B, "mu_instances": len(mu_all),
                   "steps_per_instance": n_steps, "gn_updates_per_step": 5, "modes": basis.modes(),
                   "modes_r": w.phi_r.shape[1], "n_samples": nt, "n_clusters": sur.n_clusters,
                   "n_direct": sur.n_direct, "membership_entries": int(len(L["mem_ids"])),
                   "cluster_list_entries": int(len(L["cl_list"])), "direct_list_entries": int(len(L["d_list"])),
                   "offline": offline,
                   "l2": "working set (positions of 768k sources x B instances) exceeds L2",
                   "parallelism": "single GPU" if world == 1 else f"mu instances split x{world}"},
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks.summary(),
        "finite": finite, "interactions_per_instance_step": interactions / (units * K),
    }
    defer_count(line, lambda: rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, mu_rank[:B], sys_,
                                                       pt.TimeGrid(w.dt, 1), cfg, batch=B), K * n_steps)
    return line


def _cpu_config4(w, ids, A, seconds):
    """Oracle ptrom_simulate (rom.hpp:404-412: reassign + GNAT march) for one
    μ instance over a bounded number of steps, 1 core; the surrogate build
    (offline) is excluded as in BASELINE.md §2."""
    from oracle import pyoracle
    n = w.n
    g1 = w.gamma_a + w.gamma_b
    sur = pyoracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1)
    g = w.gamma_a + float(w.mu[0]) * w.gamma_b
    t0 = time.perf_counter()
    pyoracle.ptrom_simulate(sur, w.phi, w.sv, w.x0, ids, A, g, w.delta, w.dt, 1, 1e-300, 5)
    dt1 = time.perf_counter() - t0
    steps = int(max(1, min(w.n_steps, seconds / max(dt1, 1e-6))))
    t0 = time.perf_counter()
    pyoracle.ptrom_simulate(sur, w.phi, w.sv, w.x0, ids, A, g, w.delta, w.dt, steps, 1e-300, 5)
    dt = time.perf_counter() - t0
    return {"value": steps / dt, "unit": "instance-steps/s", "cores": 1, "kind": "port",
            "sample": f"1 instance x {steps} steps (reassign + 5 GN updates/step) of config4, {dt:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference for config3 / config4: the oracle port (the reference
    does not build here), bounded sample, rank 0 only."""
    if rank != 0:
        return 0
    from oracle import pyoracle
    from paper_2103_01983_b200 import workloads
    pyoracle.build()
    K = _steps(args, 3)
    vals = []
    if args.workload == "config3":
        w = workloads.config3()
        for _ in range(K):
            vals.append(_cpu_config3(w, 0.5, 32, 8.0, threads=os.cpu_count() or 1))
        unit, metric = "bodies/s", "Barnes-Hut velocity evaluation bodies/s (fp64; build + aggregation + far field)"
    else:
        import paper_2103_01983_b200  # noqa: F401  (workload generation only)
        w = workloads.config4()
        ids = pyoracle.greedy_sample(w.phi_r, w.n_samples)
        A = pyoracle.build_gnat_operator(w.phi_r, ids)
        for _ in range(K):
            vals.append(_cpu_config4(w, ids, A, 8.0))
        unit, metric = "instance-steps/s", "PTROM online instance-steps/s (fp64)"
    value = float(np.mean([v["value"] for v in vals]))
    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": args.gpus, "steps": K, "warmup": 0,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64)", "impl": "reference", "config": {"workload": w.name},
            "cpu_baseline": {**vals[-1], "value": value},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0
