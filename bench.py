#!/usr/bin/env python3
"""bench.py — Biot–Savart pair interactions/s (fp64) on B200.

Default workload (BASELINE.json's metric configuration, configs[4]): one
all-pairs velocity evaluation of the N = 4,194,304 uniform-square system
(δ = 1e-3 → reference delta 1e-6) per step, fp64, SURVEY.md §8d config 5.
With --gpus G > 1 (torchrun, one rank per GPU) the targets are split evenly
across ranks and every step exchanges the source positions first (peer-memory
reads fused into the tile loads, or an NCCL all-gather) —
strong scaling: total work per step is fixed.

At G = 1 the line also carries the other BASELINE configs under "extra",
each with its own value, e2e, roofline, cpu_baseline and clocks:
  config1  FOM trajectory (N = 4,096, 100 steps; integrators.hpp:243-272)
  config2  single evaluation at N = 65,536, fp64 and fp32
  config3  Barnes–Hut build + aggregation + far field at N = 1,048,576
  config4  PTROM online, 4,096 μ instances x 50 steps (rom.hpp:404-412)
(--no-extras skips them; --workload configK runs one of them as the headline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload configK]

`value` is device-timed (CUDA events, max over ranks) with inputs resident in
HBM; `e2e` times the drop-in host C-ABI call (pinned host buffers in, H2D +
kernels + D2H inside the timed region). `--impl reference` times the
reference's CPU algorithm (the oracle port in oracle/, all host threads) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Biot-Savart pair interactions/s (fp64)"
UNIT = "pairs/s"
FLOPS_PER_PAIR = 12  # BASELINE.md §2 convention (kernel.hpp:33-41 + 121-122)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace('.', '', 1).isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace('.', '', 1).isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks(device: int):
    """FP64/FP32 pipe peaks measured live (tools/peaks.cu); MEASURED_PEAKS.json has HBM and bf16 only."""
    import ctypes
    lib_path = os.path.join(ROOT, "tools", "libptrom_peaks.so")
    if not os.path.exists(lib_path):
        return None
    lib = ctypes.CDLL(lib_path)
    out = (ctypes.c_double * 9)()
    if lib.ptrom_peaks(device, out) != 0:
        return None
    return {"fp64_dfma_tflops": out[0], "fp32_ffma_tflops": out[1], "mufu_rcp64h_tops": out[2],
            "dmma_fp64_tflops": out[3], "rcp_seed_max_rel_err": out[4], "rcp_newton1_max_rel_err": out[5],
            "rcp_cubic_max_rel_err": out[6]}


def ncu_traffic(name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed `ncu --set full` summary of the same kernel (profiles/)."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        d = json.load(open(path))  # written by tools/ncu_summary.py (bytes)
        return float(d["dram_bytes_per_launch"])
    except Exception:
        return None


def cpu_baseline_sample(w, threads: int, target_seconds: float, fp32: bool = False):
    """Oracle (the reference's serial loop, kernel.hpp:107-129) on a bounded
    target sample × all sources; returns pairs/s and the sample description."""
    from oracle import pyoracle
    n = w.n
    x = w.x0.astype(np.float32) if fp32 else w.x0
    g = w.gamma.astype(np.float32) if fp32 else w.gamma
    t0 = time.perf_counter()
    probe = max(8, 64 * threads)
    pyoracle.pairwise_velocity(x, g, w.delta, t_begin=0, t_end=probe, threads=threads)
    dt = time.perf_counter() - t0
    rows = int(min(n, max(probe, probe * target_seconds / max(dt, 1e-6))))
    t0 = time.perf_counter()
    pyoracle.pairwise_velocity(x, g, w.delta, t_begin=0, t_end=rows, threads=threads)
    dt = time.perf_counter() - t0
    pairs = rows * (n - 1)
    return pairs / dt, (f"{rows} targets x {n} sources of {w.name} (N={n}){' in fp32' if fp32 else ''}, "
                        f"{dt:.1f} s, {threads} thread(s)")


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port; the
    reference itself does not build here: Eigen absent)."""
    if rank != 0:
        return 0
    if args.workload == "config1":
        return run_reference_config1(args)
    if args.workload not in ("config2", "config5"):
        import bench_extra
        return bench_extra.run_reference(args, rank, world)
    from paper_2103_01983_b200 import workloads
    from oracle import pyoracle
    pyoracle.build()
    w = workloads.config5() if args.workload == "config5" else workloads.config2()
    threads = os.cpu_count() or 1
    # calibrate one step to ~1.5 s of CPU work
    t0 = time.perf_counter()
    probe = 32 * threads
    pyoracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=0, t_end=probe, threads=threads)
    rows = int(min(w.n, max(probe, probe * 1.5 / max(time.perf_counter() - t0, 1e-6))))
    for _ in range(args.warmup):
        pyoracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=0, t_end=rows, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        pyoracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=0, t_end=rows, threads=threads)
        times.append(time.perf_counter() - t0)
    pairs = rows * (w.n - 1)
    value = pairs * len(times) / sum(times)
    sample = f"{rows} targets x {w.n} sources per step ({w.name}, N={w.n}); oracle port, {threads} threads"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "impl": "reference",
        "config": {"workload": w.name, "n": w.n, "delta": w.delta, "sample_targets": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def allpairs_line(args, w, K, W, rank, world, local, e2e_steps, cpu_seconds, with_fp32, traffic_file=None):
    """One all-pairs velocity evaluation per step (kernel.hpp:107-129) of
    workload w; K timed steps after W warm-up steps (L2 flushed between)."""
    import torch
    import torch.distributed as dist

    import paper_2103_01983_b200 as pt
    from paper_2103_01983_b200 import device as dev

    n = w.n
    lo, hi = rank * n // world, (rank + 1) * n // world
    m = hi - lo
    x_full = torch.tensor(w.x0, device="cuda")
    gamma = torch.tensor(w.gamma, device="cuda")
    x_local = x_full.view(2, n)[:, lo:hi].contiguous()
    out = torch.empty(2 * m, dtype=torch.float64, device="cuda")
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    ctx = pt.default_context(local)
    stream = torch.cuda.current_stream()
    lib = ctx.lib

    ctx.set_stream(stream.cuda_stream)
    comm = None
    if world > 1:
        # the C ABI's communicator (NCCL over NVLink / NVSwitch): the exchange
        # is one grouped broadcast per rank block, then the local tile kernel
        try:
            from paper_2103_01983_b200.comm import Comm
            comm = Comm.nccl(ctx)
        except Exception as exc:  # keep torch's all-gather; the line says so
            comm_error = f"{type(exc).__name__}: {exc}"
        x_ws = torch.empty(2 * n, dtype=torch.float64, device="cuda")

    def step_allgather():  # per-evaluation exchange + local kernel (ptrom_dev_pairwise_velocity_sharded_f64)
        if comm is not None:
            ctx.check(lib.ptrom_dev_pairwise_velocity_sharded_f64(ctx.handle, comm.handle, n, x_local.data_ptr(),
                                                                  x_ws.data_ptr(), gamma.data_ptr(), w.delta, 0,
                                                                  None, out.data_ptr()))
            return
        if world > 1:
            dist.all_gather_into_tensor(x_full[:n], x_local[0])
            dist.all_gather_into_tensor(x_full[n:], x_local[1])
        dev.pairwise_velocity(x_full, gamma, w.delta, 0, None, lo, hi, out, ctx=ctx)

    # N > 1: the exchange fused into the kernel — each rank publishes its block
    # in CUDA-IPC memory and the tile loads read the peers' blocks in place over
    # NVLink (paper_2103_01983_b200/peer.py). Verified once against the
    # all-gather path; PTROM_EXCHANGE=nccl selects the all-gather path.
    if comm is not None:  # check the C-ABI path once against torch's all-gather + the one-sided kernel
        try:
            step_allgather()
            got = out.clone()
            dist.all_gather_into_tensor(x_full[:n], x_local[0])
            dist.all_gather_into_tensor(x_full[n:], x_local[1])
            dev.pairwise_velocity(x_full, gamma, w.delta, 0, None, lo, hi, out, ctx=ctx)
            dev.synchronize(ctx)
            err = float(torch.linalg.norm(got - out) / torch.linalg.norm(out))  # unordered pairs: 1e-12 parity
            ok = torch.tensor([1.0 if err <= 1e-12 else 0.0], device="cuda")
        except Exception as exc:
            comm_error = f"{type(exc).__name__}: {exc}"
            ok = torch.tensor([0.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if float(ok.item()) != 1.0:
            comm_error = locals().get("comm_error", "sharded C-ABI result differs from the all-gather path")
            comm = None
    exchange = "single-gpu"
    step = step_allgather
    if world > 1:
        exchange = (("ptrom_comm NCCL all-gather-v; unordered-pair block split + one reduce-scatter of the partial "
                     "rows" if n % world == 0 and n >= 16384 else "ptrom_comm NCCL all-gather-v")
                    if comm is not None else f"torch NCCL all-gather ({comm_error})")
        # PTROM_EXCHANGE=peer: the one-sided kernel reading the peers' blocks in place
        if os.environ.get("PTROM_EXCHANGE", "comm") == "peer" or comm is None:
            try:
                from paper_2103_01983_b200.peer import PeerExchange
                pex = PeerExchange(n, ctx)
                token = torch.zeros(1, dtype=torch.float32, device="cuda")

                def step_peer():
                    pex.write_local(x_local)
                    pex.barrier(token)  # every rank published before any rank reads
                    pex.velocity(gamma, w.delta, out)
                    pex.barrier(token)  # every rank's reads done before any rank's next write (WAR)

                step_allgather()
                ref_out = out.clone()
                step_peer()
                dev.synchronize(ctx)
                same = torch.tensor([1.0 if torch.equal(out, ref_out) else 0.0], device="cuda")
                dist.all_reduce(same, op=dist.ReduceOp.MIN)
                if float(same.item()) == 1.0:
                    exchange, step = "peer-ipc (fused into the tile loads)", step_peer
            except Exception as exc:  # keep the NCCL path; say why in the JSON line
                exchange = f"ptrom_comm NCCL all-gather-v (peer setup failed: {type(exc).__name__})"

    for _ in range(W):
        step()
    dev.synchronize(ctx)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    import ctypes
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    with ClockSampler(local) as clocks:
        lib.ptrom_profile_begin(ctx.handle)
        for k in range(K):
            l2_flush.zero_()
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        kern_ms, kern_launches = ctypes.c_double(), ctypes.c_int64()
        ctx.check(lib.ptrom_profile_end(ctx.handle, ctypes.byref(kern_ms), ctypes.byref(kern_launches)))
        torch.cuda.synchronize()
    dev.synchronize(ctx)
    step_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([step_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    pairs_per_step = n * (n - 1)
    value = pairs_per_step * K / (total_ms * 1e-3)

    # ---- e2e through the drop-in host C-ABI (pinned host buffers, H2D + D2H inside)
    if world == 1:
        hx = torch.tensor(w.x0).pin_memory().numpy()
        hg = torch.tensor(w.gamma).pin_memory().numpy()
        hf = torch.empty(2 * n, dtype=torch.float64).pin_memory().numpy()
        cnt = ctypes.c_uint64()
        fn = lambda: ctx.check(lib.ptrom_pairwise_velocity_f64(ctx.handle, n, hx.ctypes.data, hg.ctypes.data,
                                                               float(w.delta), 0, None, hf.ctypes.data,
                                                               ctypes.byref(cnt)))
        fn()  # first host-API call sizes the staging buffers
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn()
        e2e_s = time.perf_counter() - t0
        e2e = {"value": pairs_per_step * e2e_steps / e2e_s, "unit": UNIT, "steps": e2e_steps,
               "h2d_bytes_per_step": int(hx.nbytes + hg.nbytes), "d2h_bytes_per_step": int(hf.nbytes),
               "api": "ptrom_pairwise_velocity_f64 (host buffers)"}
    else:
        # Sharded end to end: every step each rank copies its own positions in
        # from pinned host memory, exchanges the sources, evaluates its
        # targets and copies its velocity rows back out (max over ranks).
        hx_local = x_local.cpu().pin_memory()
        hf_local = torch.empty(2 * m, dtype=torch.float64).pin_memory()

        def e2e_step():
            x_local.copy_(hx_local, non_blocking=True)
            step()
            hf_local.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs_per_step * e2e_steps / float(e2e_s.item()), "unit": UNIT, "steps": e2e_steps,
               "h2d_bytes_per_step": int(hx_local.numel() * 8 * world),
               "d2h_bytes_per_step": int(hf_local.numel() * 8 * world),
               "api": f"per rank: H2D own positions, {exchange}, ptrom_dev_pairwise_velocity_f64, D2H own rows"}

    if rank != 0:
        return None

    peaks = measured_peaks(local)
    avg_kernel_s = (kern_ms.value * 1e-3) / max(1, kern_launches.value)
    local_pairs = m * (n - 1)
    achieved_tf = FLOPS_PER_PAIR * local_pairs / avg_kernel_s / 1e12
    roofline = None
    if peaks:
        roofline = {"bound": "fp64", "achieved": achieved_tf, "peak": peaks["fp64_dfma_tflops"],
                    "unit": "TFLOP/s", "frac": achieved_tf / peaks["fp64_dfma_tflops"],
                    "traffic": ncu_traffic(traffic_file) if traffic_file else None,
                    "algorithmic_bytes_per_launch": 24 * n,
                    "kernel": ("allpairs_sym_kernel (csrc/allpairs_sym.cu: unordered pairs, one reciprocal per pair "
                               "for both directions)" if n >= 16384 and (world == 1 or n % world == 0)
                               else "allpairs_f64_kernel<128,8,2,1,vel> (csrc/allpairs.cu)"),
                    "peak_source": "measured live: tools/peaks.cu DFMA chain (MEASURED_PEAKS.json has no FP64)",
                    "flops_per_pair": FLOPS_PER_PAIR, "pairs_per_launch": local_pairs,
                    "avg_launch_ms": avg_kernel_s * 1e3, "launches": kern_launches.value,
                    "share_of_step": (kern_ms.value / max(1, kern_launches.value)) / (total_ms / K),
                    "peaks": peaks}

    # config 2's fp32 run (BASELINE configs[1]: "fp64 and fp32"): same workload,
    # device-timed, L2 flushed; reported beside the fp64 line
    fp32 = None
    if world == 1 and with_fp32:
        x32, g32 = x_full.float(), gamma.float()
        out32 = torch.empty(2 * n, dtype=torch.float32, device="cuda")
        for _ in range(3):
            dev.pairwise_velocity(x32, g32, w.delta, 0, None, 0, n, out32, ctx=ctx)
        torch.cuda.synchronize()
        k32 = max(10, min(K, 100))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k32)]
        with ClockSampler(local) as clocks32:
            for a, b in ev:
                l2_flush.zero_()
                a.record(stream)
                dev.pairwise_velocity(x32, g32, w.delta, 0, None, 0, n, out32, ctx=ctx)
                b.record(stream)
            torch.cuda.synchronize()
        ms32 = sum(a.elapsed_time(b) for a, b in ev) / k32
        v32 = pairs_per_step / (ms32 * 1e-3)
        hx32 = torch.tensor(w.x0, dtype=torch.float32).pin_memory().numpy()
        hg32 = torch.tensor(w.gamma, dtype=torch.float32).pin_memory().numpy()
        hf32 = torch.empty(2 * n, dtype=torch.float32).pin_memory().numpy()
        fn32 = lambda: ctx.check(lib.ptrom_pairwise_velocity_f32(ctx.handle, n, hx32.ctypes.data, hg32.ctypes.data,
                                                                 float(w.delta), 0, None, hf32.ctypes.data, None))
        fn32()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn32()
        e32 = time.perf_counter() - t0
        cpu32 = None
        if not args.no_cpu_baseline:
            v_cpu, sample = cpu_baseline_sample(w, 1, cpu_seconds / 2, fp32=True)
            cpu32 = {"value": v_cpu, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
        fp32 = {"value": v32, "unit": UNIT, "ms_per_step": ms32, "steps": k32, "dtype": "f32",
                "e2e": {"value": pairs_per_step * e2e_steps / e32, "unit": UNIT, "steps": e2e_steps,
                        "h2d_bytes_per_step": int(hx32.nbytes + hg32.nbytes), "d2h_bytes_per_step": int(hf32.nbytes),
                        "api": "ptrom_pairwise_velocity_f32 (host buffers)"},
                "roofline": {"bound": "fp32", "achieved": FLOPS_PER_PAIR * v32 / 1e12,
                             "peak": peaks["fp32_ffma_tflops"] if peaks else None, "unit": "TFLOP/s",
                             "frac": FLOPS_PER_PAIR * v32 / 1e12 / peaks["fp32_ffma_tflops"] if peaks else None,
                             "traffic": None,
                             "kernel": "allpairs_sym_f32_kernel (csrc/allpairs_sym.cu, unordered pairs), step incl. "
                                       "the block-partial reduction"},
                "cpu_baseline": cpu32, "clocks": clocks32.summary(),
                "parity": "judged against the fp64 oracle at 1e-5 (tests/test_allpairs_gpu.py)"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, sample = cpu_baseline_sample(w, 1, cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}

    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": w.name, "n": n, "delta": w.delta, "targets_per_rank": m,
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "parallelism": f"targets sharded x{world}, position exchange per step: {exchange}"
                   if world > 1 else "single GPU"},
        "gpu_launches": (kern_launches.value if world == 1 else K) * (1 if n * m <= 268435456 else 2),
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks.summary(),
        "fp32": fp32,
    }


def config1_line(args, K, W, local, cpu_seconds):
    """BASELINE configs[0]: the implicit-trapezoidal FOM trajectory
    (integrators.hpp:243-272) at N = 4,096, 100 steps, dt = 1e-3,
    NewtonConfig{1e-10, 100, 1}; one step = one whole trajectory through
    ptrom_dev_fom_simulate_f64 (device-side Newton control, CUDA graph).
    Unit: pair interactions/s counting velocity pairs (12 flops) and
    Jacobian pairs (21 flops), N(N-1) per evaluation."""
    import torch

    import paper_2103_01983_b200 as pt
    from paper_2103_01983_b200 import device as dev
    from paper_2103_01983_b200 import workloads
    w = workloads.config1()
    n = w.n
    ctx = pt.default_context(local)
    stream = torch.cuda.current_stream()
    x0 = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    snaps = torch.empty(w.n_steps, 2 * n, dtype=torch.float64, device="cuda")
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}

    def step():
        res["r"] = dev.fom_simulate(x0, g, w.delta, w.dt, w.n_steps, snapshots=snaps, ctx=ctx)

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    nv = nj = 0
    with ClockSampler(local) as clocks:
        for k in range(K):
            l2_flush.zero_()
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            nv += res["r"][4]
            nj += res["r"][5]
        torch.cuda.synchronize()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    pairs = n * (n - 1)
    value = (nv + nj) * pairs / (total_ms * 1e-3)
    flops = (12 * nv + 21 * nj) * pairs
    peaks = measured_peaks(local)
    achieved = flops / (total_ms * 1e-3) / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peaks["fp64_dfma_tflops"] if peaks else None,
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_dfma_tflops"] if peaks else None,
                "traffic": ncu_traffic("r02_fom_persistent_ncu_summary.json"),
                "kernel": "fom_persistent_kernel<256, 2> (csrc/fom_persistent.cu): the whole trajectory in one "
                          "cooperative launch",
                "scope": "whole trajectory (latency-bound at N = 4,096: two grid barriers per Newton iteration, "
                         "148 CTAs)",
                "flops_convention": "12 per velocity pair + 21 per Jacobian pair (BASELINE.md §2)",
                "velocity_evals_per_trajectory": nv / K, "jacobian_evals_per_trajectory": nj / K,
                "peak_source": "measured live: tools/peaks.cu DFMA chain"}
    # e2e: the drop-in host entry point (x0, Γ in; snapshots, iterations out)
    sys_ = pt.ParticleSystem(w.gamma, w.delta)
    grid = pt.TimeGrid(w.dt, w.n_steps)
    pt.fom_simulate(w.x0, sys_, grid)
    ke = max(3, min(K, 10))
    t0 = time.perf_counter()
    for _ in range(ke):
        run = pt.fom_simulate(w.x0, sys_, grid)
    e2e_s = time.perf_counter() - t0
    e2e = {"value": (nv + nj) / K * pairs * ke / e2e_s, "unit": UNIT, "steps": ke,
           "h2d_bytes_per_step": int(w.x0.nbytes + w.gamma.nbytes),
           "d2h_bytes_per_step": int(run.snapshots.nbytes + 13 * w.n_steps),
           "api": "ptrom_fom_simulate_f64 (host x0, Γ in; snapshots, iterations, converged, residuals out)"}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import pyoracle
        steps_cpu = w.n_steps
        t0 = time.perf_counter()
        _, it_o, _, _ = pyoracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, 10, threads=1)
        dt10 = time.perf_counter() - t0
        steps_cpu = int(min(w.n_steps, max(10, 10 * cpu_seconds / max(dt10, 1e-6))))
        t0 = time.perf_counter()
        _, it_o, _, _ = pyoracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, steps_cpu, threads=1)
        dtc = time.perf_counter() - t0
        evals = 1 + int(np.sum(it_o)) + int(np.sum(np.asarray(it_o) > 0))
        cpu = {"value": evals * pairs / dtc, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"oracle fom_simulate, {steps_cpu} of {w.n_steps} steps of {w.name} "
                         f"({evals} velocity+Jacobian evaluations, {dtc:.1f} s, 1 thread)"}
    line = {
        "metric": "Biot-Savart pair interactions/s (fp64), FOM trajectory (velocity + Jacobian pairs)",
        "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W, "ms_per_step": total_ms / K,
        "higher_is_better": True, "scaling": "weak", "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": w.name, "n": n, "delta": w.delta, "dt": w.dt, "n_steps": w.n_steps,
                   "newton": "tol 1e-10, max_iters 100, refresh 1 (integrators.hpp:55-58)",
                   "unit_of_step": "one 100-step trajectory", "l2": "flushed between trajectories"},
        "trajectory_ms": total_ms / K, "newton_updates_per_trajectory": float(np.sum(res["r"][1])),
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks.summary(),
    }
    import bench_extra
    bench_extra.defer_count(line, step, K)
    return line


def extras(args, local):
    """The other BASELINE configs at one GPU, compact runs (bounded time)."""
    import copy

    import bench_extra
    from paper_2103_01983_b200 import workloads
    out = {}
    small = copy.copy(args)
    small.cpu_seconds = min(args.cpu_seconds, 8.0)

    def guard(name, fn):
        t0 = time.perf_counter()
        try:
            out[name] = fn()
        except Exception as exc:  # an extra never hides the headline; say what failed
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        if isinstance(out[name], dict):
            out[name]["bench_seconds"] = time.perf_counter() - t0

    guard("config1", lambda: config1_line(small, 10, 3, local, small.cpu_seconds))
    guard("config2", lambda: allpairs_line(small, workloads.config2(), 20, 3, 0, 1, local, 10,
                                           small.cpu_seconds, True, "r02_allpairs_sym_c2_ncu_summary.json"))

    def c3():
        a = copy.copy(small)
        a.steps, a.steps_given, a.warmup = 10, True, 3
        line = bench_extra.bench_config3(a, 1)
        line.pop("units_per_step", None)
        return line

    def c4():
        a = copy.copy(small)
        a.steps, a.steps_given, a.warmup, a.batch = 8, True, 3, 512
        line = bench_extra.bench_config4(a, 1)
        line.pop("units_per_step", None)
        return line

    guard("config3", c3)
    guard("config4", c4)
    bench_extra.run_deferred_counts()
    return out


def run_reference_config1(args):
    """--impl reference --workload config1: the oracle's fom_simulate
    (integrators.hpp:243-272) on all host threads, a bounded number of steps
    of the config-1 trajectory per step."""
    from oracle import pyoracle
    from paper_2103_01983_b200 import workloads
    pyoracle.build()
    w = workloads.config1()
    threads = os.cpu_count() or 1
    pairs = w.n * (w.n - 1)
    vals, times = [], []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, it, _, _ = pyoracle.fom_simulate(w.x0, w.gamma, w.delta, w.dt, 10, threads=threads)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            evals = 1 + int(np.sum(it)) + int(np.sum(np.asarray(it) > 0))
            vals.append(evals * pairs)
            times.append(dt)
    value = sum(vals) / sum(times)
    sample = f"oracle fom_simulate, 10 of {w.n_steps} steps of {w.name} per step, {threads} threads"
    print(json.dumps({
        "metric": "Biot-Savart pair interactions/s (fp64), FOM trajectory (velocity + Jacobian pairs)",
        "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)", "impl": "reference",
        "config": {"workload": w.name, "n": w.n, "steps_per_sample": 10},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: 3 for config5, 200 for config2)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="config5: skip the other configs' keys")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--workload", choices=["config1", "config2", "config3", "config4", "config5"], default="config5",
                    help="config5 (default: the metric's N = 4,194,304 evaluation) | config1 FOM trajectory | "
                         "config2 N = 65,536 evaluation | config3 Barnes-Hut | config4 PTROM online batch")
    ap.add_argument("--batch", type=int, default=512, help="config4: instances per step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.steps_given = args.steps is not None
    if args.steps is None:
        args.steps = {"config5": 3, "config1": 20}.get(args.workload, 200)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.workload in ("config3", "config4"):
        import bench_extra
        if args.impl == "reference":
            return bench_extra.run_reference(args, rank, world)
        return bench_extra.run(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2103_01983_b200 import workloads

    torch.cuda.set_device(local)
    if args.workload == "config1":
        if rank == 0:
            import bench_extra
            line = config1_line(args, args.steps, args.warmup, local, args.cpu_seconds)
            bench_extra.run_deferred_counts()
            print(json.dumps(line), flush=True)
        return 0
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    big = args.workload == "config5"
    w = workloads.config5() if big else workloads.config2()
    line = allpairs_line(args, w, args.steps, args.warmup, rank, world, local,
                         2 if big else max(5, min(args.steps, 50)), args.cpu_seconds, not big,
                         "r02_allpairs_sym_c5_ncu_summary.json" if big else "r02_allpairs_sym_c2_ncu_summary.json")
    if rank == 0:
        if big and world == 1 and not args.no_extras:
            line["extra"] = extras(args, local)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
