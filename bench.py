#!/usr/bin/env python
"""Benchmark of the B200-native matrix-free operator apply.

Headline (BASELINE.json metric, config 2 = configs[1]): constant-coefficient
P1 15-point stencil apply with the full ghost-layer (interface replica) update
on the unit cube split into 6 Kuhn macro-tets at level 8 (17,173,254 slots,
16,974,593 owned DoFs), fp64, x = random_fill(seed 0). One step = one
apply (per-cell rows kernel + interface pass). Inputs (x + y = 275 MB) exceed
the 126 MB L2, so no explicit flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the macro-cells are partitioned over the ranks
(weak scaling: an N x 1 x 1 box of unit cubes, 6 Kuhn macro-tets = one
config-2-sized block per GPU, level 8). Each step is the per-cell rows
kernel on the rank's cells plus the interface exchange of the groups that
span ranks (pack, NCCL allreduce, member-order finish); times are max over
ranks. `--impl reference` times the reference CPU implementation
(oracle/_ref, the unmodified blocktet headers) on the host cores instead.
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

LEVEL = 8
WORKLOAD = "cube-kuhn (6 macro-tets) L8, P1 const-coeff 15-point stencil apply + interface sync"
METRIC = "GDoF/s of matrix-free operator apply (fp64)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0, period_ms=100):
        self.cmd = ["nvidia-smi", f"--id={index}",
                    "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                    "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                    "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                    "--format=csv,noheader,nounits", f"-lms={period_ms}"]
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(self.cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_baseline_sample(threads=None):
    """Reference CPU apply (oracle/_ref = blocktet headers, -O3, no -march),
    config 2 at full size, threads = min(#cells, nproc). Bounded sample:
    median of 5 applies (~2-10 s)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    nproc = os.cpu_count() or 1
    threads = threads or min(6, nproc)
    kind = "reference"
    try:
        r = pyoracle.Reference(pyoracle.cube_kuhn_text(), LEVEL, LEVEL)
        x = r.random_fill(LEVEL, 0)
        sec = r.time_apply(LEVEL, x, kind=0, form=0, bc=0, reps=5, threads=threads)
        owned = r.owned_count(LEVEL)
    except (FileNotFoundError, OSError):
        kind = "port"
        threads = 1
        o = pyoracle.Oracle(pyoracle.cube_kuhn_text(), LEVEL, LEVEL, with_edges=False)
        x = o.random_fill(LEVEL, 0)
        t0 = time.perf_counter()
        o.apply_stencil(LEVEL, x, 0)
        sec = time.perf_counter() - t0
        owned = o.owned_count(LEVEL)
    return {"value": owned / sec / 1e9, "unit": "GDoF/s", "cores": threads, "kind": kind,
            "sample": f"median of 5 full config-2 applies (cube-kuhn L8, {owned} owned DoFs), "
                      f"{threads} threads of {nproc} host cores, {sec * 1e3:.1f} ms/apply"}


def run_reference(args):
    """The reference CPU apply (oracle/_ref, unmodified blocktet headers) on
    the host cores, same workload/metric; rank 0 only. Each step is one full
    config-2 apply; K is capped so the run stays within about a minute."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    nproc = os.cpu_count() or 1
    threads = min(6, nproc)  # the reference parallelises over macro-cells only (threading.hpp:14)
    try:
        r = pyoracle.Reference(pyoracle.cube_kuhn_text(), LEVEL, LEVEL)
        kind = "reference"
    except (FileNotFoundError, OSError) as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    x = r.random_fill(LEVEL, 0)
    owned = r.owned_count(LEVEL)
    for _ in range(min(args.warmup, 1)):
        r.time_apply(LEVEL, x, kind=0, form=0, bc=0, reps=1, threads=threads)
    t0 = time.perf_counter()
    first = r.time_apply(LEVEL, x, kind=0, form=0, bc=0, reps=1, threads=threads)
    K = max(1, min(args.steps, int(60.0 / max(first, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(K):
        r.time_apply(LEVEL, x, kind=0, form=0, bc=0, reps=1, threads=threads)
    sec = (time.perf_counter() - t0) / K
    value = owned / sec / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": args.gpus,
            "steps": K, "warmup": min(args.warmup, 1), "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (random_fill seed 0)",
            "config": {"workload": WORKLOAD, "level": LEVEL, "cells": 6, "threads": threads},
            "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": threads, "kind": kind,
                             "sample": f"{K} full config-2 applies, {threads} threads of {nproc} host cores"},
            "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        # one rank per GPU over NCCL; BT_BENCH_BACKEND=gloo runs the same
        # protocol through host-staged collectives (code-path checks on one GPU)
        backend = os.environ.get("BT_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    import paper_2308_01792_b200 as bt
    from paper_2308_01792_b200 import _lib

    dev = torch.cuda.current_device()
    if ws > 1:
        text = bt.box_mesh_text(ws, 1, 1)
        workload = (f"{ws}x1x1 unit cubes x 6 Kuhn macro-tets ({6 * ws} cells, 6 per GPU) L8, P1 const-coeff "
                    "15-point stencil apply + interface sync (cells partitioned over ranks)")
    else:
        text, workload = bt.cube_kuhn_text(), WORKLOAD
    grid = bt.Grid(text, LEVEL, LEVEL, device=dev)
    if ws > 1:
        grid.set_partition(rank, ws)
    table = bt.compute_stencil(bt.FormId.diffusion(), grid, LEVEL)
    x = bt.allocate(bt.p1_space(), grid)
    y = bt.allocate(bt.p1_space(), grid)
    bt.random_fill(x, LEVEL, 0)
    owned = bt.owned_dof_count(x, LEVEL)  # whole job
    cs = bt.n_tet((1 << LEVEL) + 1)
    _, _, c_begin, c_end = grid.partition()
    slots = (c_end - c_begin) * cs  # this rank's slots
    L = _lib.lib
    stream = torch.cuda.current_stream()
    sp = bt.api._stream()
    xp, yp = bt.api._ptr(x.values[LEVEL]), bt.api._ptr(y.values[LEVEL])

    def step(ev=None):
        # events bracket the device work of one apply: on 1 GPU the whole
        # apply_stencil (interior kernel || fused boundary kernel incl. the
        # replica sums); on N GPUs the whole partitioned apply, exchange included
        if ev is not None:
            ev[0].record(stream)
        # N > 1: per-cell rows with the NCCL interface exchange overlapped with the interior marches
        bt.api._check(L.bt_apply_stencil(table.handle, xp, yp, 0, sp))
        if ev is not None:
            ev[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(dev)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = L.bt_launch_count()
    t_start.record(stream)
    for q in range(K):
        step(evs[q])
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = L.bt_launch_count() - launches0
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in evs]
    if ws > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / K
    value = owned * K / (total_ms * 1e-3) / 1e9
    kmean = float(np.mean(kern_ms))
    peak, peak_kind = measured_peaks()
    traffic = None  # DRAM bytes per apply from the committed ncu capture (profiles/r1_traffic.json)
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            traffic = float(json.load(f)["apply_total"]) if ws == 1 else None
    except Exception:
        traffic = None
    alg_bytes = 16.0 * slots  # read x once, write y once
    achieved = alg_bytes / (kmean * 1e-3) / 1e9

    # e2e through the public API, as a pipelined serving loop: every step
    # copies its inputs pinned host -> device and its result device -> pinned
    # host; consecutive steps overlap on three streams (H2D of step s+1, apply
    # of step s, D2H of step s-1 — PCIe is full duplex), double-buffered.
    # (per rank: its own cells' vector — a partitioned grid stores only those)
    lo, hi = 0, slots
    assert x.values[LEVEL].numel() == slots
    hx = torch.empty(slots, dtype=torch.float64, pin_memory=True)
    hx.copy_(x.values[LEVEL][lo:hi].cpu())
    hys = [torch.empty(slots, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    xs = [bt.allocate(bt.p1_space(), grid) for _ in range(2)]
    ys = [bt.allocate(bt.p1_space(), grid) for _ in range(2)]
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def serve(nsteps):
        for q in range(nsteps):
            b = q & 1
            with torch.cuda.stream(s_in):
                if q >= 2:
                    s_in.wait_event(ev_cmp[b])  # the apply of step q-2 has read xs[b]
                xs[b].values[LEVEL][lo:hi].copy_(hx, non_blocking=True)
                ev_in[b].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[b])
                if q >= 2:
                    s_cmp.wait_event(ev_out[b])  # the D2H of step q-2 has read ys[b]
                bt.apply_stencil(table, xs[b], ys[b], LEVEL)
                ev_cmp[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[b])
                hys[b].copy_(ys[b].values[LEVEL][lo:hi], non_blocking=True)
                ev_out[b].record(s_out)

    e2e_steps = max(4, min(20, K))
    serve(4)  # warm-up
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    serve(e2e_steps)
    s_out.wait_event(ev_out[(e2e_steps - 1) & 1])
    e1.record(s_out)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    hy = hys[(e2e_steps - 1) & 1]
    assert np.array_equal(hy.numpy(), y.values[LEVEL][lo:hi].cpu().numpy()), "e2e result differs from resident run"
    e2e_value = owned * e2e_steps / (e2e_ms * 1e-3) / 1e9

    if rank == 0:
        cpu = cpu_baseline_sample() if ws == 1 and not args.no_cpu else None
        line = {
            "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (random_fill seed 0, reference mt19937_64 stream)",
            "config": {"workload": workload, "level": LEVEL, "cells": grid.n_cells(), "slots_per_gpu": slots,
                       "owned_dofs": owned, "bc": "none",
                       "l2": "inputs larger than L2 (x+y = %.0f MB per GPU)" % (alg_bytes / 1e6),
                       "parallelism": f"cells partitioned over {ws} ranks, memory-sharded vectors (NCCL interface exchange)"
                       if ws > 1 else "1 GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_stencil_fast || k_boundary" if ws == 1 else "k_stencil (per-cell rows)",
                         "kernel_ms": kmean, "kernel_share": kmean / ms_step,
                         "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs (copy)",
                         "algorithmic_bytes_per_launch": alg_bytes},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GDoF/s", "h2d_bytes_per_step": 8 * slots,
                    "d2h_bytes_per_step": 8 * slots, "steps": e2e_steps,
                    "mode": "pipelined serving loop: H2D / apply / D2H of consecutive steps overlap (double-buffered)"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
