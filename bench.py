#!/usr/bin/env python
"""Benchmark of one DS-PHD/MIB filter cycle (the north-star hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfgT]

One "step" = one full cycle (predict, sort/assign, cell update, births, moments, resampling) over one
synthetic measurement grid of BASELINE configuration cfg T (2048x2048 cells, 8M persistent + 800k
birth particles; SURVEY.md 8(d) "north-star 1-GPU target").  Inputs are resident in HBM before the
timed region; L2 is flushed (256 MiB write) between timed cycles, outside the per-cycle events.
Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the tier's reference arm)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per filter cycle and particles/s at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "particles/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# Algorithmic bytes per launch of each stage: the kernel's share of SURVEY.md 8(d)'s
# A_alg = 64 nu + 32 nu_b + 56 C.  Transient arrays of this design (keys, local
# permutations, run lists) are not algorithmic and count zero.
def stage_bytes(stage: str, cfg, n_in: int) -> float:
    nu, nb, C = cfg.nu, cfg.nu_b, cfg.C
    table = {
        "predict_sort": 32.0 * nu,   # read the state (16) + write the predicted state (16); keys stay on chip
        "cells": 28.0 * C,           # meas 8 + m_F read/write 8 + occ/free 8 + counts 4
        "list_scan": 0.0,
        "pairs": 0.0,
        "resample": 32.0 * n_in,     # read the cell-ordered predicted state (16) + write the resampled state (16)
        "moments": 0.0,              # 20 B per active cell (~1 % of C): negligible
        "births": 16.0 * nb,         # write the new-born states
    }
    return table.get(stage, 0.0)


def a_alg(cfg) -> float:
    """Method-level algorithmic bytes per cycle: 64 nu + 32 nu_b + 56 C."""
    return 64.0 * cfg.nu + 32.0 * cfg.nu_b + 56.0 * cfg.C


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML (the library
    nvidia-smi reads) polled every ~0.5 ms from a thread; `nvidia-smi -lms 5` if NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nv = None
        self.lines = []              # (sm_mhz, max_mhz, {reason names})
        self.running = False

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            self.nv, self.h = nv, h
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            self.running = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "5"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nv, self.h
        while self.running:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.lines.append((sm, self.max_mhz, {n for n, bit in zip(self.NAMES, self.bits) if r & bit}))
            except Exception:
                pass
            time.sleep(0.0005)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                self.lines.append((float(parts[0]), float(parts[1]),
                                   {n for n, v in zip(self.NAMES, parts[2:6]) if v.lower().startswith("active")}))
            except ValueError:
                continue

    def wait_ready(self, timeout: float = 15.0):
        """Block until the sampler has produced its first sample."""
        t0 = time.time()
        while (self.nv is not None or self.proc is not None) and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)

    def mark(self) -> int:
        return len(self.lines)

    def stop(self, region=None) -> dict:
        if self.nv is None and self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml and nvidia-smi unavailable"]}
        time.sleep(0.01)
        if self.nv is not None:
            self.running = False
            self.t.join(timeout=1)
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        samples = list(self.lines)
        if region is not None and region[1] > region[0]:
            samples = samples[region[0]:region[1]]       # the timed cycles only
        sm = sorted(x[0] for x in samples)
        reasons = set().union(*[x[2] for x in samples]) if samples else set()
        out = {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": samples[-1][1] if samples else None,
               "reasons": sorted(reasons), "samples": len(sm),
               "source": "NVML polled every 0.5 ms" if self.nv is not None else "nvidia-smi -lms 5"}
        if region is not None:
            out["samples_in_timed_region"] = max(0, region[1] - region[0])
        return out


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ------------------------------------------------------------------------------------------ oracle timing
def oracle_sample_cfg(cfg, rows: int):
    """A bounded sample of the workload: a band of `rows` grid rows through the sensor, with the
    particle budgets scaled by the band's share of the grid."""
    from paper_1605_02406_b200 import inputs as I
    frac = rows / cfg.height
    return I.config(cfg.name, height=rows, nu=int(cfg.nu * frac), nu_b=int(cfg.nu_b * frac)), frac


def run_oracle_steps(cfg, scene, frame_fn, steps, warmup, state=None):
    import oracle
    oracle.build()
    o = oracle.Oracle(oracle.Params(width=cfg.width, height=cfg.height, nu=cfg.nu, nu_b=cfg.nu_b,
                                    cell_size=cfg.cell_size, seed=cfg.seed, **cfg.filter_params()))
    if state is not None:
        o.set_state(state["x"], state["y"], state["vx"], state["vy"], state["w_bar"], state["m_free"], state["k"])
    k0 = state["k"] if state is not None else 0
    for k in range(warmup):
        o.step(frame_fn(k0 + k), cfg.dt)
    ts = []
    for k in range(steps):
        meas = frame_fn(k0 + warmup + k)
        t0 = time.perf_counter()
        o.step(meas, cfg.dt)
        ts.append(time.perf_counter() - t0)
    return ts


def bench_reference(args, cfg):
    """The tier's reference arm: the CPU oracle as it stands, single-threaded, on a band of the
    workload (each step = one full oracle cycle on that band)."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_1605_02406_b200 import inputs as I
    band, frac = oracle_sample_cfg(cfg, args.ref_rows)
    sc = I.scene(cfg)
    r0 = cfg.height // 2 - args.ref_rows // 2

    def frame(k):
        return sc.frame(k).numpy()[r0:r0 + args.ref_rows].copy()

    with pinned_core() as core:
        ts = run_oracle_steps(band, sc, frame, args.steps, args.warmup)
    t = sum(ts) / len(ts)
    value = band.nu / t
    sample = (f"{args.ref_rows}-row band of {cfg.name} through the sensor ({band.width}x{band.height} cells, "
              f"{band.nu} + {band.nu_b} particles), {args.steps} timed oracle cycles after {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "grid": f"{cfg.width}x{cfg.height}", "nu": cfg.nu, "nu_b": cfg.nu_b,
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "pinned_core": core, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ GPU bench
def bench_ours(args, cfg):
    import numpy as np
    import torch
    rank, local_rank, world = dist_env()
    if world > 1:
        return bench_sharded(args, cfg)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_1605_02406_b200 import dog
    from paper_1605_02406_b200 import inputs as I

    cfg_r = cfg
    sc = I.scene(cfg_r)
    settle, W, K = args.settle, args.warmup, args.steps
    nframes = settle + W + K
    frames = [sc.frame(k, device=dev).contiguous() for k in range(nframes)]
    f = dog.Filter.from_config(cfg_r)
    stream = torch.cuda.current_stream()
    for k in range(settle + W):
        f.step(frames[k], cfg.dt, stream)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    clocks = ClockSampler(local_rank)
    torch.cuda.synchronize()
    clocks.start()
    clocks.wait_ready()
    time.sleep(0.05)
    m0 = clocks.mark()
    for i in range(K):
        flush.zero_()
        ev0[i].record(stream)
        f.step(frames[settle + W + i], cfg.dt, stream)
        ev1[i].record(stream)
    torch.cuda.synchronize()
    m1 = clocks.mark()
    # the timed workload as it stands right after the timed cycles (before anything else runs on this
    # filter): the state the CPU oracle is timed from, and the particle / mass counts of the roofline
    snapshot = f.get_state()
    sc_dev = dog_scalars(f)
    # continuous operation (the filter at frame rate with nothing in between): K cycles back to back, no
    # flush (the per-cycle working set, ~0.6 GB at cfg T, exceeds the 126 MB L2)
    c0 = torch.cuda.Event(enable_timing=True); c1 = torch.cuda.Event(enable_timing=True)
    flush.zero_()
    c0.record(stream)
    for i in range(K):
        f.step(frames[settle + W + i], cfg.dt, stream)
    c1.record(stream)
    torch.cuda.synchronize()
    cont_ms = c0.elapsed_time(c1) / K
    clk = clocks.stop((m0, m1))
    # per-stage times from a separate, shorter run with stage events between the kernels (the events
    # themselves break the programmatic launch overlap, so they stay out of the timed steps above)
    nprof_steps = min(K, 5)
    f.profile_begin(nprof_steps)
    for i in range(nprof_steps):
        flush.zero_()
        f.step(frames[settle + W + i], cfg.dt, stream)
    torch.cuda.synchronize()
    stages, nprof = f.profile_end()
    step_ms = sorted(ev0[i].elapsed_time(ev1[i]) for i in range(K))
    ms_mean = float(np.mean(step_ms))
    ms_max = ms_mean

    # end-to-end through the public host entry point: pinned host meas in, host occupancy out
    e2e = None
    if args.e2e_steps > 0:
        host_frames = [frames[settle + W + (i % K)].cpu().pin_memory() for i in range(min(args.e2e_steps, K))]
        occ_host = [torch.empty(cfg.C, dtype=torch.float32).pin_memory() for _ in range(2)]
        # synchronous entry (copy in, cycle, copy out, wait) -- device-timed
        f.step_host(host_frames[0], cfg.dt, occ_host[0], stream)   # warm the staging buffer
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(args.e2e_steps):
            f.step_host(host_frames[i % len(host_frames)], cfg.dt, occ_host[0], stream)
        s1.record(stream)
        torch.cuda.synchronize()
        sync_ms = s0.elapsed_time(s1) / args.e2e_steps
        # pipelined entry: the next frame's upload and the last occupancy's download overlap the cycle;
        # host wall clock over the whole run including the final synchronisation
        f.step_host_async(host_frames[0], cfg.dt, occ_host[0], stream)
        f.sync(stream)
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            f.step_host_async(host_frames[i % len(host_frames)], cfg.dt, occ_host[i % 2], stream)
        f.sync(stream)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        # the PCIe floor: the same bytes as a bare pinned host -> device copy, back to back
        dev_buf = torch.empty_like(host_frames[0], device=dev)
        for _ in range(3):
            dev_buf.copy_(host_frames[0], non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for i in range(args.e2e_steps):
            dev_buf.copy_(host_frames[i % len(host_frames)], non_blocking=True)
        torch.cuda.synchronize()
        h2d_ms = (time.perf_counter() - t1) * 1e3 / args.e2e_steps
        del dev_buf
        # the full readout (occupied / free mass, velocity mean and covariance: 28 B per cell) every cycle
        outs = [{"occ": torch.empty(cfg.C, dtype=torch.float32).pin_memory(),
                 "free": torch.empty(cfg.C, dtype=torch.float32).pin_memory(),
                 "mean": torch.empty(cfg.C, 2, dtype=torch.float32).pin_memory(),
                 "cov": torch.empty(cfg.C, 3, dtype=torch.float32).pin_memory()} for _ in range(2)]
        f.step_host_readout(host_frames[0], cfg.dt, outs[0], stream)
        f.sync(stream)
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            f.step_host_readout(host_frames[i % len(host_frames)], cfg.dt, outs[i % 2], stream)
        f.sync(stream)
        full_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        e2e = {"value": cfg.nu / (full_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * cfg.C, "d2h_bytes_per_step": 28 * cfg.C,
               "ms_per_step": full_ms, "steps": args.e2e_steps,
               "entry": "dog_step_host_readout (pinned host meas -> device on a copy stream, cycle, the full readout "
                        "occ + free + mean + cov -> pinned host on a second copy stream; overlapped across cycles; "
                        "wall clock incl. final sync)",
               "h2d_floor_ms": h2d_ms,
               "occupancy_only": {"value": cfg.nu / (e2e_ms * 1e-3), "ms_per_step": e2e_ms,
                                  "h2d_bytes_per_step": 8 * cfg.C, "d2h_bytes_per_step": 4 * cfg.C,
                                  "entry": "dog_step_host_async"},
               "sync_entry_ms_per_step": sync_ms,
               "note": "pipelined e2e is bound by PCIe: 32 MB up and 117 MB down per cycle at cfg T (h2d_floor_ms: "
                       "the upload alone as a bare pinned copy); the cycle itself is ms_per_step"}

    # NEXT-1 (Doppler / association branch): cycles with a radar overlay on half the occupied cells,
    # device-timed like the main line (L2 flushed between cycles); continues the same filter
    doppler = None
    try:
        nd = min(K, 10)
        dops = [sc.doppler(settle + W + i, frames[settle + W + i], frac=0.5, p_assoc=0.8, sd=0.25, device=dev)
                for i in range(nd)]
        for i in range(2):
            f.step_doppler(frames[settle + W + i], dops[i][0], dops[i][1], cfg.dt, stream)
        torch.cuda.synchronize()
        d0 = [torch.cuda.Event(enable_timing=True) for _ in range(nd)]
        d1 = [torch.cuda.Event(enable_timing=True) for _ in range(nd)]
        for i in range(nd):
            flush.zero_()
            d0[i].record(stream)
            f.step_doppler(frames[settle + W + i], dops[i][0], dops[i][1], cfg.dt, stream)
            d1[i].record(stream)
        torch.cuda.synchronize()
        dms = float(np.mean([d0[i].elapsed_time(d1[i]) for i in range(nd)]))
        dop_bytes = a_alg(cfg) + 20.0 * cfg.C                  # + the Doppler grid (16 B + p_A 4 B per cell)
        doppler = {"ms_per_step": dms, "value": cfg.nu / (dms * 1e-3), "unit": UNIT,
                   "doppler_cells": int(sum(int((d[1] > 0).sum()) for d in dops) / nd),
                   "algorithmic_bytes": dop_bytes, "achieved_GBps": dop_bytes / (dms * 1e-3) / 1e9,
                   "frac": dop_bytes / (dms * 1e-3) / 1e9 / peaks()[0],
                   "input": "radar overlay on 50 % of the occupied cells, p_A 0.8, sd 0.25 m/s (inputs.Scene.doppler)"}
    except Exception as exc:   # noqa: BLE001
        doppler = {"error": str(exc)}

    # NEXT-3 (exact PHD/MIB, uniform likelihood): cycles from observation grids of the same frames,
    # device-timed like the main line; births go to every cell (r_b > 0 everywhere), so the active-cell
    # list holds the whole grid
    exact = None
    try:
        ne = min(K, 6)
        obs = [I.Scene.exact_obs(frames[settle + W + i]) for i in range(ne)]
        for i in range(12):                                # to the exact filter's steady state (spread births)
            f.step_exact(obs[i % ne], cfg.dt, stream)
        torch.cuda.synchronize()
        x0 = [torch.cuda.Event(enable_timing=True) for _ in range(ne)]
        x1 = [torch.cuda.Event(enable_timing=True) for _ in range(ne)]
        for i in range(ne):
            flush.zero_()
            x0[i].record(stream)
            f.step_exact(obs[i], cfg.dt, stream)
            x1[i].record(stream)
        torch.cuda.synchronize()
        xms = float(np.mean([x0[i].elapsed_time(x1[i]) for i in range(ne)]))
        ex_bytes = a_alg(cfg) + 16.0 * cfg.C               # obs grid is 16 B per cell instead of 8
        exact = {"ms_per_step": xms, "value": cfg.nu / (xms * 1e-3), "unit": UNIT,
                 "algorithmic_bytes": ex_bytes, "achieved_GBps": ex_bytes / (xms * 1e-3) / 1e9,
                 "frac": ex_bytes / (xms * 1e-3) / 1e9 / peaks()[0],
                 "input": "inputs.Scene.exact_obs of the same frames (DESIGN.md A-37 recipe)"}
    except Exception as exc:   # noqa: BLE001
        exact = {"error": str(exc)}

    # NEXT-3 general form: the exact filter with a single-object likelihood (A-38), continuing from there
    exact_lik = None
    try:
        nl = min(K, 6)
        kk = [settle + W + i for i in range(nl)]
        ins = [sc.exact_lik(k, frames[k].cpu()) for k in kk]
        ins = [tuple(t.to(dev).contiguous() for t in x) for x in ins]
        for i in range(4):
            f.step_exact_lik(*ins[i % nl], cfg.dt, stream)
        torch.cuda.synchronize()
        l0 = [torch.cuda.Event(enable_timing=True) for _ in range(nl)]
        l1 = [torch.cuda.Event(enable_timing=True) for _ in range(nl)]
        for i in range(nl):
            flush.zero_()
            l0[i].record(stream)
            f.step_exact_lik(*ins[i], cfg.dt, stream)
            l1[i].record(stream)
        torch.cuda.synchronize()
        lms = float(np.mean([l0[i].elapsed_time(l1[i]) for i in range(nl)]))
        n_lik = int(sum(((x[2] > 0) & (x[0][..., 0] > 0)).sum().item() for x in ins) / nl)
        # + lik grid 16 B and p_A 4 B per cell; members' g / gfx written and read (16 B) per particle
        lk_bytes = a_alg(cfg) + 36.0 * cfg.C + 16.0 * cfg.nu
        exact_lik = {"ms_per_step": lms, "value": cfg.nu / (lms * 1e-3), "unit": UNIT,
                     "algorithmic_bytes": lk_bytes, "achieved_GBps": lk_bytes / (lms * 1e-3) / 1e9,
                     "frac": lk_bytes / (lms * 1e-3) / 1e9 / peaks()[0], "likelihood_cells": n_lik,
                     "input": "inputs.Scene.exact_lik of the same frames (DESIGN.md A-38 recipe: radar overlay on 50 % "
                              "of the cells with a return, p_A 0.8, sd 0.25 m/s, p_cl 0.02)"}
    except Exception as exc:   # noqa: BLE001
        exact_lik = {"error": str(exc)}

    # NEXT-2 (ego-motion compensation): one scroll of grid and particles at this size, device-timed
    ego = None
    try:
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        n_ego = 6
        e0.record(stream)
        for i in range(n_ego):
            f.ego_scroll(0.35 if i % 2 == 0 else -0.35, 0.15 if i % 2 == 0 else -0.15, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ego_ms = e0.elapsed_time(e1) / n_ego
        ego_bytes = 32.0 * cfg.nu + 8.0 * cfg.C              # particles read + written, m_F read + written
        hbm0, _ = peaks()
        ego = {"ms": ego_ms, "algorithmic_bytes": ego_bytes, "achieved_GBps": ego_bytes / (ego_ms * 1e-3) / 1e9,
               "frac": ego_bytes / (ego_ms * 1e-3) / 1e9 / hbm0, "shift_cells": [3, 1]}
    except Exception as exc:   # noqa: BLE001 -- reported, not fatal to the main line
        ego = {"error": str(exc)}

    # NEXT-4 (evaluation workload): Mahalanobis per cell, 64 ROC thresholds, cluster sums -- device-timed
    evaluation = None
    try:
        labels = torch.ones(cfg.C, dtype=torch.uint8, device=dev)
        mask = torch.zeros(cfg.C, dtype=torch.uint8, device=dev)
        mask[: cfg.C // 100] = 1
        thr = np.logspace(-3, 3, 64).astype(np.float32)
        m_buf = torch.empty(cfg.C, dtype=torch.float32, device=dev)
        for _ in range(3):                                                        # warm
            f.evaluate(labels=labels, mask=mask, thresholds=thr, stream=stream, fetch=False, m=m_buf)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):    # one kernel per call; readouts (4M cells, 109 MB/pass) do not fit the L2
            f.evaluate(labels=labels, mask=mask, thresholds=thr, stream=stream, fetch=False, m=m_buf)
        e1.record(stream)
        torch.cuda.synchronize()
        ev_ms = e0.elapsed_time(e1) / reps
        t0 = time.perf_counter()
        r = f.evaluate(labels=labels, mask=mask, thresholds=thr, stream=stream, m=m_buf)
        api_ms = (time.perf_counter() - t0) * 1e3
        # algorithmic bytes per cell: mean 8 + cov 12 + label 1 + mask 1 + moments bit 1/8 read, m 4 written
        ev_bytes = (8 + 12 + 1 + 1 + 0.125 + 4) * cfg.C
        evaluation = {"ms": ev_ms, "api_ms_with_readback": api_ms, "algorithmic_bytes": ev_bytes,
                      "thresholds": 64, "achieved_GBps": ev_bytes / (ev_ms * 1e-3) / 1e9,
                      "frac": ev_bytes / (ev_ms * 1e-3) / 1e9 / peaks()[0],
                      "labelled_cells": int(r["counts"][0].sum())}
    except Exception as exc:   # noqa: BLE001
        evaluation = {"error": str(exc)}

    # per-stage times and roofline of the dominant kernel
    st_avg = {k: v / max(nprof, 1) for k, v in stages.items()}
    kern = {k: v for k, v in st_avg.items() if k != "memset"}
    dom = max(kern, key=kern.get)
    hbm, peak_src = peaks()
    bytes_dom = stage_bytes(dom, cfg, sc_dev["n_in"])
    achieved = bytes_dom / (kern[dom] * 1e-3) / 1e9
    traffic = ncu_traffic(dom)
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": bytes_dom, "avg_launch_ms": kern[dom]}
    step_roof = {"A_alg_bytes": a_alg(cfg), "achieved": a_alg(cfg) / (ms_mean * 1e-3) / 1e9,
                 "frac": a_alg(cfg) / (ms_mean * 1e-3) / 1e9 / hbm, "unit": "GB/s",
                 "formula": "64 nu + 32 nu_b + 56 C (SURVEY.md 8(d))"}

    # the other BASELINE configurations on this GPU (cfg2, cfg3, cfg5, and cfg4's 32M particles on one
    # GPU): ms per cycle, particles/s and the step roofline, timed like the main line (shorter)
    configs = run_config_lines(args, dev, stream, flush) if args.config_lines not in ("", "none") else None

    cpu = None
    if args.cpu_baseline_steps > 0:
        with pinned_core() as core:
            ts = run_oracle_steps(cfg, sc, lambda k: sc.frame(k).numpy(), args.cpu_baseline_steps, 0, state=snapshot)
        t = sum(ts) / len(ts)
        cpu = {"value": cfg.nu / t, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{len(ts)} full {cfg.name} cycles ({cfg.width}x{cfg.height}, {cfg.nu} + {cfg.nu_b}) from "
                         f"the state the GPU reached right after its timed cycles, single-threaded C oracle "
                         f"(gcc -O2 -ffp-contract=off) pinned to one core", "ms_per_step": t * 1e3,
               "pinned_core": core, "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    value = cfg.nu / (ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded ray-cast urban scene, inputs.py)",
        "config": {"workload": f"{cfg.name}: {cfg.width}x{cfg.height} grid, {cfg.nu} persistent + {cfg.nu_b} birth "
                               f"particles, urban ray-cast scene", "grid": f"{cfg.width}x{cfg.height}", "nu": cfg.nu,
                   "nu_b": cfg.nu_b, "dt_s": cfg.dt, "settle_cycles": settle,
                   "l2": "flushed between timed cycles (256 MiB write outside the cycle events)",
                   "parallelism": "single GPU",
                   "p10_p90_ms": [step_ms[int(0.1 * (K - 1))], step_ms[int(0.9 * (K - 1))]]},
        "roofline": roof, "step_roofline": step_roof,
        "stages_ms": {k: round(v, 5) for k, v in st_avg.items()},
        "cpu_baseline": cpu, "e2e": e2e,
        "continuous": {"ms_per_step": cont_ms, "value": cfg.nu / (cont_ms * 1e-3), "unit": UNIT,
                       "note": "K cycles back to back, no flush between them (working set > L2)"},
        "gpu_launches": f.launches_per_step() * K, "clocks": clk,
        "next_rows": {"doppler": doppler, "exact_phd_mib": exact, "exact_lik": exact_lik, "ego_scroll": ego, "evaluate": evaluation},
        "configs": configs,
        "n_in": sc_dev["n_in"], "W_total_mass": sc_dev["W"] * 2.0 ** -40,
        "paper_context": "GTX980: 2e6 particles, 1.44e6 cells -> 31.055 ms (PAPER.md:1832), not this workload",
    }
    print(json.dumps(line), flush=True)


def bench_sharded(args, cfg):
    """N > 1: the cfg's single scene split into N row bands, one per rank; migrants by
    NCCL send/recv between neighbour ranks, born mass and joint weight by NCCL all-gathers.  Strong
    scaling: value = the scene's nu / cycle time, the time being the max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist.init_process_group("nccl", device_id=dev)
    from paper_1605_02406_b200 import inputs as I
    from paper_1605_02406_b200 import shard

    sc = I.scene(cfg)
    settle, W, K = args.settle, args.warmup, args.steps
    t = shard.DistTransport(rank, world, dev)
    f = shard.ShardedFilter.from_config(cfg, rank, world, t)
    bands = [f.band_of(sc.frame(k, device=dev).contiguous()).contiguous() for k in range(settle + W + K)]
    stream = torch.cuda.current_stream()
    for k in range(settle + W):
        f.step(bands[k], cfg.dt, stream)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.wait_ready()
    dist.barrier()
    torch.cuda.synchronize()
    time.sleep(0.05)
    m0 = clocks.mark()
    for i in range(K):
        flush.zero_()
        ev0[i].record(stream)
        f.step(bands[settle + W + i], cfg.dt, stream)
        ev1[i].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop((m0, clocks.mark()))
    dist.barrier()
    step_ms = sorted(ev0[i].elapsed_time(ev1[i]) for i in range(K))
    ms_all = torch.tensor([float(np.mean(step_ms))], device=dev, dtype=torch.float64)
    dist.all_reduce(ms_all, op=dist.ReduceOp.MAX)
    ms_max = float(ms_all.item())
    n_own = torch.tensor([f.f.particles()[0].shape[0]], device=dev, dtype=torch.int64)
    own_all = torch.zeros(world, device=dev, dtype=torch.int64)
    dist.all_gather(list(own_all.chunk(world)), n_own)

    # end to end: the band's measurement from pinned host memory, the cycle, the band's occupancy back
    e2e = None
    if args.e2e_steps > 0:
        host = [bands[settle + W + (i % K)].cpu().pin_memory() for i in range(min(args.e2e_steps, K))]
        occ_host = torch.empty(f.f.C, dtype=torch.float32).pin_memory()
        dist.barrier()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(args.e2e_steps):
            m = host[i % len(host)].to(dev, non_blocking=True)
            f.step(m, cfg.dt, stream)
            occ_host.copy_(f.f.read_cells(stream)["occ"], non_blocking=True)
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_t = torch.tensor([s0.elapsed_time(s1) / args.e2e_steps], device=dev, dtype=torch.float64)
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.nu / (float(e2e_t.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * cfg.C, "d2h_bytes_per_step": 4 * cfg.C,
               "ms_per_step": float(e2e_t.item()), "steps": args.e2e_steps,
               "entry": "BandFilter phases per rank (pinned host band meas -> device, cycle, band occupancy -> host)"}
    hbm, peak_src = peaks()
    per_gpu = a_alg(cfg) / world / (ms_max * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": cfg.nu / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded ray-cast urban scene, inputs.py)",
            "config": {"workload": f"{cfg.name}: {cfg.width}x{cfg.height} grid, {cfg.nu} persistent + {cfg.nu_b} "
                                   f"birth particles, urban ray-cast scene", "grid": f"{cfg.width}x{cfg.height}",
                       "nu": cfg.nu, "nu_b": cfg.nu_b, "dt_s": cfg.dt, "settle_cycles": settle,
                       "l2": "flushed between timed cycles (256 MiB write outside the cycle events)",
                       "parallelism": f"row bands x{world} (migrants: owner buckets, NCCL send/recv + all-gather; "
                                      f"prefixes: NCCL all-gather)",
                       "rows": shard.band_rows(cfg.height, world), "own_particles": own_all.tolist(),
                       "p10_p90_ms": [step_ms[int(0.1 * (K - 1))], step_ms[int(0.9 * (K - 1))]]},
            "roofline": {"bound": "hbm", "kernel": "cycle per GPU (A_alg / N)", "achieved": per_gpu, "peak": hbm,
                         "unit": "GB/s", "frac": per_gpu / hbm, "traffic": None, "peak_source": peak_src},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": 11 * K * world, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


class pinned_core:
    """Context manager: run on one host core (the first this process may use), as `taskset -c` would."""
    def __enter__(self):
        self.prev = None
        try:
            self.prev = os.sched_getaffinity(0)
            core = min(self.prev)
            os.sched_setaffinity(0, {core})
            return core
        except Exception:   # noqa: BLE001 -- not Linux: unpinned
            return None

    def __exit__(self, *exc):
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)
        return False


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:   # noqa: BLE001
        pass
    return "unknown"


def run_config_lines(args, dev, stream, flush):
    """ms per cycle, particles/s and the step roofline of the other BASELINE configurations on one GPU."""
    import numpy as np
    import torch
    from paper_1605_02406_b200 import dog
    from paper_1605_02406_b200 import inputs as I
    hbm, _ = peaks()
    out = {}
    for name in args.config_lines.split(","):
        if name == args.config or name not in I.CONFIGS:
            continue
        try:
            cfg = I.CONFIGS[name]
            sc = I.scene(cfg)
            settle, K = 30, 8
            frames = [sc.frame(k, device=dev).contiguous() for k in range(settle + K)]
            f = dog.Filter.from_config(cfg)
            for k in range(settle):
                f.step(frames[k], cfg.dt, stream)
            torch.cuda.synchronize()
            e0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
            e1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
            for i in range(K):
                flush.zero_()
                e0[i].record(stream)
                f.step(frames[settle + i], cfg.dt, stream)
                e1[i].record(stream)
            torch.cuda.synchronize()
            ms = float(np.mean([e0[i].elapsed_time(e1[i]) for i in range(K)]))
            A = a_alg(cfg)
            out[name] = {"workload": f"{cfg.width}x{cfg.height} grid, {cfg.nu} + {cfg.nu_b} particles",
                         "ms_per_step": ms, "value": cfg.nu / (ms * 1e-3), "unit": UNIT,
                         "particles_incl_births_per_s": (cfg.nu + cfg.nu_b) / (ms * 1e-3),
                         "step_roofline": {"A_alg_bytes": A, "achieved": A / (ms * 1e-3) / 1e9,
                                           "frac": A / (ms * 1e-3) / 1e9 / hbm},
                         "steps": K, "settle_cycles": settle}
            f.close()
            del frames, f
            torch.cuda.empty_cache()
        except Exception as exc:   # noqa: BLE001
            out[name] = {"error": str(exc)}
    return out


def dog_scalars(f):
    import numpy as np
    from paper_1605_02406_b200 import dog
    a = np.zeros(8, np.uint64)
    rc = dog.dog_get_debug(f.handle, dog.DEBUG_IDS["SCALARS"], a.ctypes.data, a.nbytes)
    if rc < 0:
        return {"n_in": 0, "W": 0}
    return {"n_in": int(a[7]), "W": int(a[0])}


def ncu_traffic(kernel_stage: str):
    """DRAM bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel_stage)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfgT")
    ap.add_argument("--settle", type=int, default=30, help="untimed cycles from the empty state before warm-up")
    ap.add_argument("--e2e-steps", type=int, default=60)
    ap.add_argument("--cpu-baseline-steps", type=int, default=2)
    ap.add_argument("--ref-rows", type=int, default=256)
    ap.add_argument("--config-lines", default="cfg2,cfg3,cfg5,cfg4",
                    help="other configurations timed on this GPU (comma-separated; empty: none)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    from paper_1605_02406_b200 import inputs as I
    cfg = I.CONFIGS[args.config]
    if args.impl == "reference":
        bench_reference(args, cfg)
    else:
        bench_ours(args, cfg)


if __name__ == "__main__":
    main()
