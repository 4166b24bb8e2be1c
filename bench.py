#!/usr/bin/env python3
"""bench.py — Biot–Savart pair interactions/s (fp64) on B200.

Workload (BASELINE.json configs[1]): one all-pairs velocity evaluation of the
N = 65,536 Gaussian vortex patch (δ = 0.005 → reference delta 2.5e-5) per
step, fp64, SURVEY.md §8d. With --gpus G > 1 (torchrun, one rank per GPU)
the targets are split evenly across ranks and every step all-gathers the
source positions over NCCL first (the per-evaluation exchange of the sharded
FOM) — strong scaling: total work per step is fixed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value` is device-timed (CUDA events, max over ranks) with inputs resident in
HBM; `e2e` times the drop-in host C-ABI call (ptrom_pairwise_velocity_f64:
pinned host buffers in, H2D + kernels + D2H inside the timed region).
`--impl reference` times the reference's CPU algorithm (the oracle port in
oracle/, all host threads) on a bounded sample of the same workload.
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


def cpu_baseline_sample(w, threads: int, target_seconds: float):
    """Oracle (the reference's serial loop, kernel.hpp:107-129) on a bounded
    target sample × all sources; returns pairs/s and the sample description."""
    from oracle import pyoracle
    n = w.n
    t0 = time.perf_counter()
    probe = max(8, 64 * threads)
    pyoracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=0, t_end=probe, threads=threads)
    dt = time.perf_counter() - t0
    rows = int(min(n, max(probe, probe * target_seconds / max(dt, 1e-6))))
    t0 = time.perf_counter()
    pyoracle.pairwise_velocity(w.x0, w.gamma, w.delta, t_begin=0, t_end=rows, threads=threads)
    dt = time.perf_counter() - t0
    pairs = rows * (n - 1)
    return pairs / dt, f"{rows} targets x {n} sources of {w.name} (N={n}), {dt:.1f} s"


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port; the
    reference itself does not build here: Eigen absent)."""
    if rank != 0:
        return 0
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: 200 for config2)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--workload", choices=["config2", "config3", "config4", "config5"], default="config2",
                    help="config2 (default, the headline) | config3 Barnes-Hut | config4 PTROM online batch | "
                         "config5 all-pairs evaluation at N = 4,194,304 (the 8-GPU sharded config)")
    ap.add_argument("--batch", type=int, default=512, help="config4: instances per step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.steps_given = args.steps is not None
    if args.steps is None:
        args.steps = 3 if args.workload == "config5" else 200
    if args.workload not in ("config2", "config5"):
        import bench_extra
        rank = env_int("RANK", 0)
        world = env_int("WORLD_SIZE", 1)
        if args.impl == "reference":
            return bench_extra.run_reference(args, rank, world)
        return bench_extra.run(args, rank, world)

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2103_01983_b200 as pt
    from paper_2103_01983_b200 import device as dev
    from paper_2103_01983_b200 import workloads

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workloads.config5() if args.workload == "config5" else workloads.config2()
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

    def step_allgather():  # per-evaluation exchange: NCCL all-gather of the positions, then the local kernel
        if world > 1:
            dist.all_gather_into_tensor(x_full[:n], x_local[0])
            dist.all_gather_into_tensor(x_full[n:], x_local[1])
        dev.pairwise_velocity(x_full, gamma, w.delta, 0, None, lo, hi, out, ctx=ctx)

    # N > 1: the exchange fused into the kernel — each rank publishes its block
    # in CUDA-IPC memory and the tile loads read the peers' blocks in place over
    # NVLink (paper_2103_01983_b200/peer.py). Verified once against the
    # all-gather path; PTROM_EXCHANGE=nccl selects the all-gather path.
    exchange = "single-gpu"
    step = step_allgather
    if world > 1:
        exchange = "nccl-allgather"
        if os.environ.get("PTROM_EXCHANGE", "peer") == "peer":
            try:
                from paper_2103_01983_b200.peer import PeerExchange
                pex = PeerExchange(n, ctx)
                token = torch.zeros(1, dtype=torch.float32, device="cuda")

                def step_peer():
                    pex.write_local(x_local)
                    pex.barrier(token)
                    pex.velocity(gamma, w.delta, out)

                step_allgather()
                ref_out = out.clone()
                step_peer()
                dev.synchronize(ctx)
                same = torch.tensor([1.0 if torch.equal(out, ref_out) else 0.0], device="cuda")
                dist.all_reduce(same, op=dist.ReduceOp.MIN)
                if float(same.item()) == 1.0:
                    exchange, step = "peer-ipc (fused into the tile loads)", step_peer
            except Exception as exc:  # keep the NCCL path; say why in the JSON line
                exchange = f"nccl-allgather (peer setup failed: {type(exc).__name__})"

    for _ in range(args.warmup):
        step()
    dev.synchronize(ctx)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    lib = ctx.lib
    with ClockSampler(local) as clocks:
        lib.ptrom_profile_begin(ctx.handle)
        for k in range(args.steps):
            l2_flush.zero_()
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        import ctypes
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
    value = pairs_per_step * args.steps / (total_ms * 1e-3)

    # ---- e2e through the drop-in host C-ABI (pinned host buffers, H2D + D2H inside)
    e2e = None
    if world == 1:
        hx = torch.tensor(w.x0).pin_memory().numpy()
        hg = torch.tensor(w.gamma).pin_memory().numpy()
        hf = torch.empty(2 * n, dtype=torch.float64).pin_memory().numpy()
        sys_ = pt.ParticleSystem(hg, w.delta)
        import ctypes
        cnt = ctypes.c_uint64()
        fn = lambda: ctx.check(lib.ptrom_pairwise_velocity_f64(ctx.handle, n, hx.ctypes.data, hg.ctypes.data,
                                                               float(w.delta), 0, None, hf.ctypes.data,
                                                               ctypes.byref(cnt)))
        big = args.workload == "config5"  # ~10 s per evaluation
        for _ in range(1 if big else 3):
            fn()
        e2e_steps = max(1, args.steps) if big else max(5, min(args.steps, 50))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn()
        e2e_s = time.perf_counter() - t0
        e2e = {"value": pairs_per_step * e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(hx.nbytes + hg.nbytes), "d2h_bytes_per_step": int(hf.nbytes),
               "api": "ptrom_pairwise_velocity_f64 (host buffers)"}
        del sys_
    else:
        # Sharded end to end: every step each rank copies its own positions in
        # from pinned host memory, all-gathers the sources, evaluates its
        # targets and copies its velocity rows back out (max over ranks).
        hx_local = x_local.cpu().pin_memory()
        hf_local = torch.empty(2 * m, dtype=torch.float64).pin_memory()
        e2e_steps = max(5, min(args.steps, 50))

        def e2e_step():
            x_local.copy_(hx_local, non_blocking=True)
            step()
            hf_local.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(3):
            e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs_per_step * e2e_steps / float(e2e_s.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(hx_local.numel() * 8 * world),
               "d2h_bytes_per_step": int(hf_local.numel() * 8 * world),
               "api": "per rank: H2D own positions, NCCL all-gather, ptrom_dev_pairwise_velocity_f64, D2H own rows"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = measured_peaks(local)
    avg_kernel_s = (kern_ms.value * 1e-3) / max(1, kern_launches.value)
    local_pairs = m * (n - 1)
    achieved_tf = FLOPS_PER_PAIR * local_pairs / avg_kernel_s / 1e12
    roofline = None
    if peaks:
        roofline = {"bound": "fp64", "achieved": achieved_tf, "peak": peaks["fp64_dfma_tflops"],
                    "unit": "TFLOP/s", "frac": achieved_tf / peaks["fp64_dfma_tflops"],
                    "traffic": ncu_traffic("r01_allpairs_vel64_ncu_summary.json") if args.workload == "config2" else None,
                    "algorithmic_bytes_per_launch": 24 * n,
                    "kernel": "allpairs_f64_kernel<128,8,2,1,vel> (csrc/allpairs.cu)",
                    "peak_source": "measured live: tools/peaks.cu DFMA chain (MEASURED_PEAKS.json has no FP64)",
                    "flops_per_pair": FLOPS_PER_PAIR, "pairs_per_launch": local_pairs,
                    "avg_launch_ms": avg_kernel_s * 1e3, "launches": kern_launches.value,
                    "peaks": peaks}

    # config 2's fp32 run (BASELINE configs[1]: "fp64 and fp32"): same workload,
    # device-timed, L2 flushed; reported beside the fp64 headline
    fp32 = None
    if world == 1 and args.workload == "config2":
        x32, g32 = x_full.float(), gamma.float()
        out32 = torch.empty(2 * n, dtype=torch.float32, device="cuda")
        for _ in range(3):
            dev.pairwise_velocity(x32, g32, w.delta, 0, None, 0, n, out32, ctx=ctx)
        torch.cuda.synchronize()
        k32 = max(10, min(args.steps, 100))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k32)]
        for a, b in ev:
            l2_flush.zero_()
            a.record(stream)
            dev.pairwise_velocity(x32, g32, w.delta, 0, None, 0, n, out32, ctx=ctx)
            b.record(stream)
        torch.cuda.synchronize()
        ms32 = sum(a.elapsed_time(b) for a, b in ev) / k32
        v32 = pairs_per_step / (ms32 * 1e-3)
        fp32 = {"value": v32, "unit": UNIT, "ms_per_step": ms32, "steps": k32,
                "roofline": {"bound": "fp32", "achieved": FLOPS_PER_PAIR * v32 / 1e12,
                             "peak": peaks["fp32_ffma_tflops"] if peaks else None, "unit": "TFLOP/s",
                             "frac": FLOPS_PER_PAIR * v32 / 1e12 / peaks["fp32_ffma_tflops"] if peaks else None,
                             "kernel": "allpairs_f32_kernel<128,8> (csrc/allpairs.cu), step incl. chunk reduction"}}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, sample = cpu_baseline_sample(w, 1, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": w.name, "n": n, "delta": w.delta, "targets_per_rank": m,
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "parallelism": f"targets sharded x{world}, position exchange per step: {exchange}"
                   if world > 1 else "single GPU"},
        "gpu_launches": 2 * args.steps,  # tile kernel + fixed-order chunk reduction
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks.summary(),
        "fp32": fp32,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
