#!/usr/bin/env python
"""MCI benchmark (BASELINE.json metric: output samples/s (fp32) and achieved HBM GB/s).

Default workload = BASELINE.json configs[1] ("config 2"): 65536 real signals,
M=3 channels (f, f', f''), N=1024 samples each -> L=16384 outputs, fp32.
A step is one pass of the whole hot path (forward DFTs, per-class solves,
assembly, inverse FFTs, stores) over the batch, i.e. one mci_execute_1d.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..9] [--impl mci|reference]

N > 1: one process per GPU (torchrun), each rank runs its own batch (rows are
independent: weak scaling, no collective on the data path); time = max over
ranks of the CUDA-event time.  Rank 0 prints ONE JSON line.
--impl reference times the fp64 CPU oracle (the tier's reference arm) on a
bounded sample on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "MCI output samples/sec (fp32) and achieved HBM GB/s vs B200 peak"
UNIT = "samples/s"
# FP64 FMA throughput measured on this pool's B200 (tools/microbench/f64_throughput.cu, 1965 MHz;
# profiles/r01/microbench_f64.txt): the "alu" roofline peak of the off-grid evaluator (config 7)
FP64_PEAK_TFLOPS = 33.24


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth, burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload(cfg):
    c = synth.CONFIGS[cfg]
    if cfg == 5:
        n = c["N"]
        return dict(name=f"cfg5: {c['batch']} images, 4 channel images 512x512 -> 2048x2048 (separable, bank {{1,ik}}^2)",
                    units=c["batch"], outs_per_unit=c["size"] ** 2, in_per_unit=4 * n * n,
                    out_floats_per_unit=c["size"] ** 2)
    if cfg == 8:
        H, W, s = c["H"], c["W"], c["scale"]
        return dict(name=f"cfg8: {c['batch']} images {H}x{W} -> {s * H}x{s * W} (SISR x{s}: centred differences, "
                         f"bank 1, ik, -k^2, rows then columns; NEXT-2)",
                    units=c["batch"], outs_per_unit=s * H * s * W, in_per_unit=H * W, out_floats_per_unit=s * H * s * W)
    if cfg == 9:
        return dict(name=f"cfg9: eps(f, N) of {c['batch']} spectra x {c['nfreq']} coefficients, M={c['M']}, "
                         f"N={c['N']}, bank 1, ik, -k^2 (NEXT-4; unit = spectral coefficients)",
                    units=c["batch"], outs_per_unit=c["nfreq"], in_per_unit=2 * c["nfreq"], out_floats_per_unit=3)
    if cfg == 7:
        return dict(name=f"cfg7: {c['batch']} x (M={c['M']}, N={c['N']}) -> {c['npts']} arbitrary points x 1 out, "
                         f"bank 1, ik, -k^2 (NEXT-3 off-grid)",
                    units=c["batch"], outs_per_unit=c["npts"], in_per_unit=c["M"] * c["N"],
                    out_floats_per_unit=c["npts"])
    M, N, L, B = c["M"], c["N"], c["L"], c["batch"]
    nout = 2 if c.get("hilbert") else 1
    bank = {1: "1, ik", 2: "1, ik, -k^2", 3: "1, ik (+Hf)", 4: "delays 2 pi m/(4N)", 6: "1, ik, -k^2 (NEXT-1, odd band)"}[cfg]
    return dict(name=f"cfg{cfg}: {B} x (M={M}, N={N}) -> L={L} x {nout} out, bank {bank}",
                units=B, outs_per_unit=L * nout, in_per_unit=M * N, out_floats_per_unit=L * nout)


def make_inputs(cfg, rank):
    """Host inputs of the configuration (seeded; rank-offset seeds for N>1)."""
    c = synth.CONFIGS[cfg]
    if cfg == 1:
        return synth.cfg1(seed=rank)["g"]
    if cfg == 2:
        return synth.cfg2_batch_fast(c["batch"], seed=2 + 1000 * rank)
    if cfg == 3:
        return synth.cfg3_rows(np.arange(c["batch"]), seed=3 + 1000 * rank)
    if cfg == 4:
        return synth.cfg4_signals(np.arange(c["batch"]), seed=4 + 1000 * rank)[0]
    if cfg == 6:
        return synth.cfg2_batch_fast(c["batch"], seed=6 + 1000 * rank, M=c["M"], N=c["N"], bank=c["bank"])
    if cfg == 7:
        return synth.cfg2_batch_fast(c["batch"], seed=7 + 1000 * rank, M=c["M"], N=c["N"], bank=c["bank"])
    if cfg == 9:
        return synth.error_spectra(c["batch"], -(c["M"] * c["N"]) * 2, c["nfreq"], seed=9 + 1000 * rank)
    if cfg == 8:  # 4 distinct images tiled to the batch (content does not change the arithmetic)
        lr, _ = synth.sisr_images(range(4 * rank, 4 * rank + 4))
        return np.ascontiguousarray(np.tile(lr, (c["batch"] // 4, 1, 1)))
    # cfg5: generate a few distinct images and tile them to the batch (content does not
    # change the arithmetic or the bytes; generation of 64 2048^2 images would dominate)
    distinct = 4
    g, _ = synth.cfg5_images(range(rank * distinct, rank * distinct + distinct))
    reps = c["batch"] // distinct
    return np.ascontiguousarray(np.tile(g, (reps, 1, 1, 1, 1)))


def algorithmic_flops(cfg):
    """Algorithmic flops per unit (row / signal / image), SURVEY.md §8(d) counting."""
    c = synth.CONFIGS[cfg]
    lg = math.log2
    if cfg == 5:
        n, L = c["N"], c["N"] * c["scale"]
        line = 2 * 2.5 * n * lg(n) + 8 * 4 * (n // 2 + 1) + 2.5 * L * lg(L)
        return (2 * n + L) * line  # per image: column pass Mx*Nx = 2n lines, row pass Ly = L lines
    if cfg == 9:  # per spectrum: |a|^2 and three weighted sums per coefficient (fp64), plus the
        # per-coefficient weights (M^2 complex multiply-adds + norms), computed once per call
        return c["nfreq"] * 9 + c["nfreq"] * (8 * c["M"] ** 2 + 6 * c["M"]) / c["batch"]
    if cfg == 8:  # per image: H row lines (3 channels, N = W -> sW), then sW column lines
        H, W, s = c["H"], c["W"], c["scale"]

        def line(n, L):
            return 3 * 2.5 * n * lg(n) + 8 * 9 * (n // 2 + 1) + 2.5 * L * lg(L)
        return H * line(W, s * W) + s * W * line(H, s * H)
    M, N, L = c["M"], c["N"], c["L"]
    if cfg == 7:  # forward + solve, then a complex multiply-add per band term per point
        return M * 2.5 * N * lg(N) + 8 * M * M * (N // 2 + 1) + c["npts"] * (M * N // 2) * 8
    inv = 5 * L * lg(L) if c.get("hilbert") else 2.5 * L * lg(L)
    return M * 2.5 * N * lg(N) + 8 * M * M * (N // 2 + 1) + inv


def max_over_ranks(x: float, dist, device) -> float:
    """Max of a per-rank scalar over all ranks (the step time of a weak-scaling run)."""
    import torch
    t = torch.tensor([x], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_plan(cfg):
    import paper_1802_10291_b200 as mci
    c = synth.CONFIGS[cfg]
    if cfg == 5:
        return mci.Plan2D(2, c["N"], c["bank"], 2, c["N"], c["bank"], c["scale"])
    if cfg == 8:
        return mci.SisrPlan(c["H"], c["W"], c["scale"])
    if cfg == 9:
        return mci.Plan(c["M"], c["N"], c["L"], c["bank"], analysis=True)
    return mci.Plan(c["M"], c["N"], c["L"], c["bank"], dtype="f64" if cfg == 1 else "f32",
                    hilbert=bool(c.get("hilbert")), offgrid=cfg == 7)


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def oracle_sample(cfg, budget_s=12.0, max_steps=None):
    """Time the fp64 oracle on a bounded sample of the workload on the host cores.
    Returns (samples_per_s, description, threads, per-step seconds list)."""
    import oracle
    c = synth.CONFIGS[cfg]
    threads = os.cpu_count() or 1
    if cfg == 4:
        M, N, L = c["M"], c["N"], c["L"]
        g, _ = synth.cfg4_signals([0])
        pts = np.random.default_rng(0).integers(0, L, 64)
        t0 = time.perf_counter()
        n = 0
        while True:
            oracle.delay_eval_points(M, N, L, g[0], pts, threads=threads)
            n += len(pts)
            if time.perf_counter() - t0 > budget_s / 2:
                break
        dt = time.perf_counter() - t0
        return n / dt, f"signal 0, {n} output points (closed-form delay kernel), M*N={M*N} terms each", threads
    if cfg == 9:
        P9 = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=threads)
        s9 = make_inputs(9, 0)[:8]
        t0 = time.perf_counter()
        n = 0
        while n < len(s9):
            oracle.averaged_error(P9, s9[n].astype(np.complex128), -(c["M"] * c["N"]) * 2)
            n += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return n * c["nfreq"] / dt, f"{n} spectra x {c['nfreq']} coefficients (direct loops)", threads
    if cfg == 8:
        lr, _ = synth.sisr_images([0])
        t0 = time.perf_counter()
        n = 0
        while True:
            oracle.sisr(lr[0].astype(np.float64), c["scale"])
            n += 1
            if time.perf_counter() - t0 > budget_s / 2:
                break
        dt = time.perf_counter() - t0
        return n * (c["scale"] ** 2) * c["H"] * c["W"] / dt, f"{n} image(s) {c['H']}x{c['W']} -> x{c['scale']}", threads
    if cfg == 7:
        P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=threads)
        g = make_inputs(7, 0)[:64].astype(np.float64)
        t = synth.offgrid_points(c["npts"]).astype(np.float32).astype(np.float64)
        rows = 0
        t0 = time.perf_counter()
        while rows < len(g):
            P.eval_offgrid(g[rows], t)
            rows += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return rows * c["npts"] / dt, f"{rows} rows x {c['npts']} off-grid points (direct band sums)", threads
    if cfg == 5:
        px = oracle.OraclePlan(2, c["N"], c["N"] * c["scale"], c["bank"], threads=threads)
        px.kernel_table()
        g, _ = synth.cfg5_images([0])
        cols = np.arange(0, 2048, 2048 // 16)
        t0 = time.perf_counter()
        oracle.eval_2d_columns(g[0], px, px, cols)
        dt = time.perf_counter() - t0
        return len(cols) * 2048 / dt, f"image 0, {len(cols)} full output columns (2048 px each)", threads
    M, N, L = c["M"], c["N"], c["L"]
    P = oracle.OraclePlan(M, N, L, c["bank"], threads=threads)
    P.kernel_table()
    if c.get("hilbert"):
        P.kernel_table(True)
    rows = 0
    t0 = time.perf_counter()
    while True:
        g = make_row(cfg, rows)
        P.eval(g)
        if c.get("hilbert"):
            P.eval(g, hilbert=True)
        rows += 1
        if time.perf_counter() - t0 > budget_s or (max_steps and rows >= max_steps):
            break
    dt = time.perf_counter() - t0
    nout = 2 if c.get("hilbert") else 1
    return rows * L * nout / dt, f"{rows} rows of the workload (kernel table built before timing)", threads


def make_row(cfg, r):
    if cfg == 1:
        return synth.cfg1()["g"]
    if cfg == 2:
        return synth.cfg2_rows([r])
    if cfg == 6:
        c = synth.CONFIGS[6]
        return synth.cfg2_batch_fast(256, seed=6, M=c["M"], N=c["N"], bank=c["bank"])[r % 256][None]
    return synth.cfg3_rows([r])


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    cfg = args.config
    c = synth.CONFIGS[cfg]
    w = workload(cfg)
    threads = os.cpu_count() or 1
    # each step = one row (cfg1-3, 6), 64 points (cfg4) or 4 columns (cfg5) of the workload
    if cfg in (1, 2, 3, 6):
        P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=threads)
        P.kernel_table()
        if c.get("hilbert"):
            P.kernel_table(True)
        nout = 2 if c.get("hilbert") else 1

        def step(i):
            g = make_row(cfg, i)
            P.eval(g)
            if c.get("hilbert"):
                P.eval(g, hilbert=True)
            return c["L"] * nout
        sample = "one row per step"
    elif cfg == 4:
        gg, _ = synth.cfg4_signals([0])
        pts = np.random.default_rng(0).integers(0, c["L"], 64)

        def step(i):
            oracle.delay_eval_points(c["M"], c["N"], c["L"], gg[0], pts, threads=threads)
            return len(pts)
        sample = "64 output points of signal 0 per step (closed-form delay kernel)"
    elif cfg == 9:
        P9 = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=threads)
        s9 = make_inputs(9, 0)[:4]

        def step(i):
            oracle.averaged_error(P9, s9[i % 4].astype(np.complex128), -(c["M"] * c["N"]) * 2)
            return c["nfreq"]
        sample = "one spectrum per step (direct loops of Eq. averageerror)"
    elif cfg == 8:
        lr8, _ = synth.sisr_images([0])

        def step(i):
            oracle.sisr(lr8[0].astype(np.float64), c["scale"])
            return (c["scale"] ** 2) * c["H"] * c["W"]
        sample = "one image per step"
    elif cfg == 7:
        P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=threads)
        g7 = make_inputs(7, 0)[:64].astype(np.float64)
        t7 = synth.offgrid_points(c["npts"]).astype(np.float32).astype(np.float64)

        def step(i):
            P.eval_offgrid(g7[i % len(g7)], t7)
            return c["npts"]
        sample = f"one row's {c['npts']} off-grid points per step (direct band sums)"
    else:
        px = oracle.OraclePlan(2, c["N"], c["N"] * c["scale"], c["bank"], threads=threads)
        px.kernel_table()
        gi, _ = synth.cfg5_images([0])

        def step(i):
            oracle.eval_2d_columns(gi[0], px, px, [(i * 131) % 2048, (i * 131 + 1) % 2048])
            return 2 * 2048
        sample = "two full output columns of image 0 per step"
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    done = 0
    for i in range(args.steps):
        done += step(i)
    dt = time.perf_counter() - t0
    v = done / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": w["name"], "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def load_traffic(workload_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(workload_name)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5, 6, 7, 8, 9])
    ap.add_argument("--impl", default="mci", choices=["mci", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1802_10291_b200 as mci

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    w = workload(cfg)
    tdt = torch.float64 if cfg == 1 else torch.float32
    esz = 8 if cfg == 1 else 4

    g_host = make_inputs(cfg, rank)
    plan = make_plan(cfg)
    g = torch.from_numpy(g_host).to("cuda", dtype=torch.complex64 if cfg == 9 else tdt)
    units = w["units"]
    c = synth.CONFIGS[cfg]
    hilbert = bool(c.get("hilbert"))
    tpts = None
    if cfg == 5:
        out = torch.empty((units, c["size"], c["size"]), dtype=tdt, device="cuda")
        hf = None
    elif cfg == 8:
        out = torch.empty((units, c["scale"] * c["H"], c["scale"] * c["W"]), dtype=tdt, device="cuda")
        hf = None
    elif cfg == 9:
        out = torch.empty((units, 3), dtype=tdt, device="cuda")
        hf = None
    elif cfg == 7:
        t_host = synth.offgrid_points(c["npts"], seed=7 + 1000 * rank).astype(np.float32)
        tpts = torch.from_numpy(t_host).cuda()
        out = torch.empty((units, c["npts"]), dtype=tdt, device="cuda")
        hf = None
    else:
        out = torch.empty((units, c["L"]), dtype=tdt, device="cuda")
        hf = torch.empty_like(out) if hilbert else None
    stream = torch.cuda.current_stream()

    def step():
        if cfg in (5, 8):
            plan.execute(g, out)
        elif cfg == 7:
            plan.execute_offgrid(g, tpts, out)
        elif cfg == 9:
            plan.averaged_error(g, -(c["M"] * c["N"]) * 2, out)
        else:
            plan.execute(g, out, hf)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        ms = max_over_ranks(ms, dist, "cuda")
    ms_step = ms / args.steps
    total_samples = units * w["outs_per_unit"] * world
    value = total_samples / (ms_step / 1e3)

    # roofline of the dominant kernel: algorithmic bytes per launch / launch time.
    # (cfg2: one fused launch per step, so the kernel time is the step time on the stream.)
    peak, peak_src = load_peaks()
    launches = plan.launches(units)
    if cfg == 9:  # mci_averaged_error: the per-call weight table, then the per-spectrum sums
        launches = 2
    alg_bytes = units * (w["in_per_unit"] + w["out_floats_per_unit"]) * esz
    per_launch_ms = ms_step / launches if cfg in (1, 2, 3, 6) else ms_step
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9 if cfg in (1, 2, 3, 6) else alg_bytes / (ms_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": load_traffic(w["name"]), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes if cfg in (1, 2, 3, 6) else None,
            "algorithmic_bytes_per_step": alg_bytes}
    if cfg == 7:  # direct band sums in fp64: bound by the FP64 FMA pipe
        fl = algorithmic_flops(cfg) * units / (ms_step / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": fl, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": fl / FP64_PEAK_TFLOPS, "traffic": load_traffic(w["name"]),
                "peak_source": "measured FP64 DFMA throughput (tools/microbench/f64_throughput.cu, "
                               "profiles/r01/microbench_f64.txt)",
                "hbm_gbs_algorithmic": achieved}
    # secondary ceiling: the FP32 pipe.  Algorithmic flops per unit =
    # SURVEY.md §8(d) counts (2.5 n log2 n per real FFT, 5 n log2 n complex, 8 M^2 per class).
    flops = algorithmic_flops(cfg) * units
    sm_clock = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
    fp32_peak = 148 * 128 * 2 * sm_clock / 1e12
    roof["fp32"] = {"achieved_tflops": flops / (ms_step / 1e3) / 1e12, "peak_tflops": fp32_peak,
                    "frac": flops / (ms_step / 1e3) / 1e12 / fp32_peak,
                    "peak_source": "148 SM x 128 FP32 lanes x 2 flop x sampled SM clock"}

    # end-to-end through the host-buffer C-ABI call (H2D + compute + D2H inside)
    e2e = None
    if not args.no_e2e:
        gh = torch.from_numpy(g_host).to(torch.complex64 if cfg == 9 else tdt).pin_memory()
        oh = torch.empty(out.shape, dtype=tdt).pin_memory()
        hh = torch.empty(out.shape, dtype=tdt).pin_memory() if hilbert else None
        e_steps = max(3, min(args.steps, 10))

        if cfg == 7:
            th = torch.from_numpy(t_host).pin_memory()

        def estep():
            if cfg == 5:
                plan.execute_host(gh, oh)
            elif cfg == 9:  # public device API with the host copies inside the timed step
                oh.copy_(plan.averaged_error(gh.to("cuda", non_blocking=True), -(c["M"] * c["N"]) * 2),
                         non_blocking=True)
                torch.cuda.synchronize()
            elif cfg == 8:  # public device API with the host copies inside the timed step
                oh.copy_(plan.execute(gh.to("cuda", non_blocking=True)), non_blocking=True)
                torch.cuda.synchronize()
            elif cfg == 7:  # public device API with the host copies inside the timed step
                gd = gh.to("cuda", non_blocking=True)
                td = th.to("cuda", non_blocking=True)
                oh.copy_(plan.execute_offgrid(gd, td), non_blocking=True)
                torch.cuda.synchronize()
            else:
                plan.execute_host(gh, oh, hh)
        estep()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            estep()
        et = (time.perf_counter() - t0) / e_steps
        if world > 1:
            et = max_over_ranks(et, dist, "cuda")
        e2e = {"value": total_samples / et, "unit": UNIT,
               "h2d_bytes_per_step": int(gh.numel() * esz) + (int(th.numel() * esz) if cfg == 7 else 0),
               "d2h_bytes_per_step": int(oh.numel() * esz * (2 if hilbert else 1)),
               "ms_per_step": et * 1e3, "steps": e_steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample, thr = oracle_sample(cfg)
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64" if cfg == 1 else "f32",
                "data": "synthetic",
                "config": {"workload": w["name"], "units_per_gpu": units,
                           "l2": "inputs+outputs exceed the 126 MB L2 (no flush needed)" if cfg != 1 else
                           "tiny (latency-bound), L2-resident",
                           "parallelism": f"dp{world} (independent rows per rank)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches * args.steps),
                "clocks": clk.summary(),
                "hbm_gbs_algorithmic": achieved}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
