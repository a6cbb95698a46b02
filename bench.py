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
    bank = {1: "1, ik", 2: "1, ik, -k^2", 3: "1, ik (+Hf)", 4: "delays 2 pi m/(4N)", 6: "1, ik, -k^2 (NEXT-1, odd band)",
            10: "1, ik (off-benchmark shape)", 11: "1, ik, -k^2, -ik^3 (off-benchmark shape)",
            12: "8 interleaved delays 2 pi m/(MN) (off-benchmark shape)"}[cfg]
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
    if cfg in (6, 10, 11, 12):
        return synth.cfg2_batch_fast(c["batch"], seed=cfg + 1000 * rank, M=c["M"], N=c["N"], bank=c["bank"])
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class OracleLeg:
    """The fp64 oracle on units of the benchmarked workload itself (rows / points / columns /
    images / spectra of the same seeded inputs): its plan is built once (reported separately),
    then each sampled unit is evaluated, timed, and kept so that the GPU's outputs for the same
    units can be compared afterwards (the bench line's parity and cpu_baseline come from one
    run of the oracle)."""

    def __init__(self, cfg, g_host, tpts=None, rank=0, threads=None):
        import oracle
        self.oracle = oracle
        self.cfg, self.g, self.tpts = cfg, g_host, tpts
        self.c = c = synth.CONFIGS[cfg]
        self.threads = threads or (os.cpu_count() or 1)
        self.rank = rank
        t0 = time.perf_counter()
        if cfg in (1, 2, 3, 6, 7, 10, 11, 12):
            self.P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=self.threads)
            if cfg != 7:
                self.P.kernel_table()
                if c.get("hilbert"):
                    self.P.kernel_table(True)
        elif cfg == 5:
            self.P = oracle.OraclePlan(2, c["N"], c["N"] * c["scale"], c["bank"], threads=self.threads)
            self.P.kernel_table()
        elif cfg == 9:
            self.P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"], threads=self.threads)
        self.plan_s = time.perf_counter() - t0
        # unit order: spread over the batch (the first and last units included)
        self.order = {2: _spread(c.get("batch", 1), 4096), 3: _spread(c.get("batch", 1), 512),
                      10: _spread(c.get("batch", 1), 2048), 11: _spread(c.get("batch", 1), 4096),
                      12: _spread(c.get("batch", 1), 4096),
                      6: _spread(c.get("batch", 1), 4096), 7: _spread(c.get("batch", 1), 512),
                      8: _spread(c.get("batch", 1), 64), 9: _spread(c.get("batch", 1), 512)}.get(cfg)
        if cfg == 4:
            self.pts = np.random.default_rng(0).choice(c["L"], 1 << 16, replace=False)
        if cfg == 5:
            self.cols = np.random.default_rng(0).permutation(c["size"])
        self.results = []  # (unit key, oracle output)

    def set_threads(self, n):
        self.threads = n
        if hasattr(self, "P"):
            self.P.threads = n

    def unit(self, i):
        """Evaluate sampled unit i; returns (key, oracle values, output samples)."""
        o, c, cfg = self.oracle, self.c, self.cfg
        if cfg == 1:
            return 0, self.P.eval(self.g), c["L"]
        if cfg in (2, 6, 10, 11, 12):
            r = int(self.order[i % len(self.order)])
            return r, self.P.eval(self.g[r:r + 1])[0], c["L"]
        if cfg == 3:
            r = int(self.order[i % len(self.order)])
            return r, (self.P.eval(self.g[r:r + 1])[0], self.P.eval(self.g[r:r + 1], hilbert=True)[0]), 2 * c["L"]
        if cfg == 4:  # 64 output points of signal 0 per unit (closed-form delay kernel)
            p = self.pts[64 * (i % 1024): 64 * (i % 1024) + 64]
            return tuple(p), o.delay_eval_points(c["M"], c["N"], c["L"], self.g[0], p, threads=self.threads), len(p)
        if cfg == 5:  # two full output columns of image 0 per unit
            cols = self.cols[2 * (i % 1024): 2 * (i % 1024) + 2]
            return tuple(cols), o.eval_2d_columns(self.g[0], self.P, self.P, cols), 2 * c["size"]
        if cfg == 7:
            r = int(self.order[i % len(self.order)])
            return r, self.P.eval_offgrid(self.g[r], self.tpts.astype(np.float64)), c["npts"]
        if cfg == 8:
            r = int(self.order[i % len(self.order)])
            return r, o.sisr(self.g[r].astype(np.float64), c["scale"], threads=self.threads), \
                (c["scale"] ** 2) * c["H"] * c["W"]
        r = int(self.order[i % len(self.order)])  # cfg 9
        k_lo = -(c["M"] * c["N"]) * 2
        return r, np.array(o.averaged_error(self.P, self.g[r].astype(np.complex128), k_lo)), c["nfreq"]

    def run(self, budget_s, max_units=None, keep=True):
        """Evaluate units until budget_s; returns (samples per second, units done)."""
        done = n = 0
        t0 = time.perf_counter()
        while True:
            key, val, outs = self.unit(n)
            if keep:
                self.results.append((key, val))
            done += outs
            n += 1
            if time.perf_counter() - t0 > budget_s or (max_units and n >= max_units) or self.cfg == 1:
                break
        return done / (time.perf_counter() - t0), n

    def sample_text(self, n):
        c, cfg = self.c, self.cfg
        return {1: "the whole workload (one fp64 row)",
                2: f"{n} rows spread over the batch", 3: f"{n} rows spread over the batch (f and Hf)",
                4: f"{64 * n} output points of signal 0 (closed-form delay kernel, {c.get('M', 0) * c.get('N', 0)} "
                   f"terms each)",
                5: f"{2 * n} full output columns of image 0", 6: f"{n} rows spread over the batch",
                10: f"{n} rows spread over the batch", 11: f"{n} rows spread over the batch",
                12: f"{n} rows spread over the batch",
                7: f"{n} rows x {c.get('npts')} off-grid points (direct band sums)",
                8: f"{n} image(s) {c.get('H')}x{c.get('W')} -> x{c.get('scale')}",
                9: f"{n} spectra x {c.get('nfreq')} coefficients (direct loops)"}[cfg] + \
            " (oracle plan / kernel tables built before timing)"

    def parity(self, out, hf=None):
        """Per-unit relative L2 error of the GPU outputs of the sampled units."""
        import torch
        rel = []
        for key, val in self.results:
            if self.cfg == 1:
                got = out[0].double().cpu().numpy()
                rel.append(_rel(got, val[0]))
            elif self.cfg == 3:
                rel.append(_rel(out[key].double().cpu().numpy(), val[0]))
                rel.append(_rel(hf[key].double().cpu().numpy(), val[1]))
            elif self.cfg == 4:
                idx = torch.tensor(key, device=out.device)
                rel.append(_rel(out[0, idx].double().cpu().numpy(), val))
            elif self.cfg == 5:
                idx = torch.tensor(key, device=out.device)
                rel.append(_rel(out[0][:, idx].double().cpu().numpy(), val))
            elif self.cfg == 9:
                got = out[key].double().cpu().numpy()
                rel.append(float(np.max(np.abs(got - val) / np.abs(val))))
            else:
                rel.append(_rel(out[key].double().cpu().numpy(), val))
        return np.asarray(rel)


def _spread(batch, n):
    n = min(n, batch)
    mid = np.random.default_rng(12345).permutation(np.arange(1, max(batch - 1, 1)))[: max(n - 2, 0)]
    return np.concatenate([[0], [batch - 1] if batch > 1 else [], mid]).astype(np.int64)


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_reference(args, rank, world):
    """--impl reference: the tier's reference arm is the fp64 oracle (the paper ships no code),
    timed as it stands on the host cores, one sampled unit of the same workload per step."""
    if rank != 0:
        return
    cfg = args.config
    w = workload(cfg)
    g_host = make_inputs(cfg, 0)
    tpts = synth.offgrid_points(synth.CONFIGS[7]["npts"], seed=7).astype(np.float32) if cfg == 7 else None
    leg = OracleLeg(cfg, g_host, tpts)
    for i in range(args.warmup):
        leg.unit(i)
    t0 = time.perf_counter()
    done = 0
    for i in range(args.steps):
        done += leg.unit(args.warmup + i)[2]
    dt = time.perf_counter() - t0
    v = done / dt
    sample = leg.sample_text(1).replace(" (oracle plan", " per step (oracle plan")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": w["name"], "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": leg.threads, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model(), "plan_s": leg.plan_s},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def load_traffic(workload_name):
    """ncu DRAM bytes (read + write) for this workload, from the committed capture summary
    (profiles/ncu_traffic.json, written by tools/ncu_summarize.py): per step (all launches of
    one step) when a step-wide metrics capture exists, else per launch of the dominant kernel.
    Returns (bytes, scope, source) or (None, None, None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh).get(workload_name)
    except Exception:
        return None, None, None
    if d is None:
        return None, None, None
    if isinstance(d, dict):
        return d.get("bytes"), d.get("scope"), d.get("source")
    return d, "dominant kernel, one launch", "profiles/ncu_traffic.json"


def load_inst(workload_name):
    """ncu-counted warp instructions of one step (smsp__inst_executed.sum over the step's MCI
    launches) from profiles/ncu_traffic.json, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh).get(workload_name)
    except Exception:
        return None
    if isinstance(d, dict) and d.get("inst"):
        return {"inst": d["inst"], "source": d.get("source")}
    return None


def relaunch_cmd(args_list, n, port):
    """The torchrun command that runs this script on n ranks of one node (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(args_list)


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def dry_run_gloo(args, rank, world):
    """CPU check of the multi-rank host path (tests/test_multirank.py): the torchrun
    relaunch, the gloo rendezvous, per-rank seeded inputs, the max-over-ranks step time
    and the single JSON line of rank 0.  No GPU work."""
    import torch.distributed as dist
    dist.init_process_group("gloo")
    g = make_inputs(1, rank)
    ms = max_over_ranks(1.0 + rank, dist, "cpu")
    digests = [None] * world
    dist.all_gather_object(digests, float(np.abs(g).sum()))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ms_per_step": ms,
                          "distinct_inputs": len(set(digests)) == world}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=list(range(1, 13)))
    ap.add_argument("--impl", default="mci", choices=["mci", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run-gloo", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched as plain `python bench.py --gpus N`: one process per GPU under torchrun
        if not args.dry_run_gloo:
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible")
        import subprocess
        sys.exit(subprocess.call(relaunch_cmd(sys.argv[1:], args.gpus, free_port())))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run_gloo:
        dry_run_gloo(args, rank, world)
        return

    import torch
    import torch.distributed as dist

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
    tpts = t_host = None
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
    k_lo9 = -(c.get("M", 0) * c.get("N", 0)) * 2

    def step():
        if cfg in (5, 8):
            plan.execute(g, out)
        elif cfg == 7:
            plan.execute_offgrid(g, tpts, out)
        elif cfg == 9:
            plan.averaged_error(g, k_lo9, out)
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
    # (configs 1-3, 6, 9: one launch per step, so the kernel time is the step time on the stream;
    #  configs 4, 5, 8: several kernels per step, so the step's algorithmic bandwidth.)
    peak, peak_src = load_peaks()
    launches = plan.launches(units)
    alg_bytes = units * (w["in_per_unit"] + w["out_floats_per_unit"]) * esz
    if cfg == 9:  # the method reads only the out-of-band coefficients (in-band ones carry no error)
        alg_bytes = units * ((c["nfreq"] - c["M"] * c["N"]) * 2 * esz + w["out_floats_per_unit"] * esz)
    single = cfg in (1, 2, 3, 6, 9, 10, 11, 12)
    achieved = alg_bytes / (ms_step / 1e3) / 1e9
    tr_bytes, tr_scope, tr_src = load_traffic(w["name"])
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": tr_bytes, "traffic_scope": tr_scope, "traffic_source": tr_src, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes if single else None,
            "algorithmic_bytes_per_step": alg_bytes,
            "scope": "single kernel (one launch per step)" if single else f"step ({launches} launches)"}
    if cfg == 9:
        roof["bytes_note"] = "out-of-band coefficients (8 B each) + 3 outputs per spectrum; in-band ones are not read"
    if cfg == 7:  # direct band sums in fp64: bound by the FP64 FMA pipe
        fl = algorithmic_flops(cfg) * units / (ms_step / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": fl, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": fl / FP64_PEAK_TFLOPS, "traffic": tr_bytes, "traffic_scope": tr_scope,
                "traffic_source": tr_src,
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
    # instruction-issue ceiling (the kernels of configs 6-8 are issue-bound by construction, so
    # their HBM fraction says little): ncu-counted warp instructions of one step (committed
    # launch list) over this run's step time, vs 148 SM x 4 schedulers x 1 warp-instr/clk
    inst = load_inst(w["name"])
    if inst:
        ach = inst["inst"] / (ms_step / 1e3) / 1e9
        peak_i = 148 * 4 * sm_clock / 1e9
        roof["issue"] = {"achieved_ginst_s": ach, "peak_ginst_s": peak_i, "frac": ach / peak_i,
                         "inst_per_step": inst["inst"], "source": inst["source"],
                         "peak_source": "148 SM x 4 schedulers x 1 warp instruction / clk x sampled SM clock"}

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
                oh.copy_(plan.averaged_error(gh.to("cuda", non_blocking=True), k_lo9), non_blocking=True)
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
        del gh, oh, hh

    # quality numbers BASELINE.json names for the configuration (not timed)
    quality = quality_numbers(cfg, out, hf, rank)

    # cpu_baseline (rank 0, N = 1): the oracle as it stands on units of this same workload,
    # and the parity of the GPU outputs for those units
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        leg = OracleLeg(cfg, g_host, t_host, rank)
        v, n = leg.run(12.0)
        leg.set_threads(1)
        v1, n1 = leg.run(4.0, max_units=max(1, n // 4), keep=False)
        cpu = {"value": v, "unit": UNIT, "cores": (os.cpu_count() or 1), "kind": "oracle",
               "sample": leg.sample_text(n), "cpu_model": cpu_model(),
               "single_thread_value": v1, "single_thread_sample": f"{n1} unit(s), threads=1",
               "plan_s": leg.plan_s,
               "full_config_s_extrapolated": leg.plan_s + units * w["outs_per_unit"] / v}
        rel = leg.parity(out, hf)
        tol = 1e-11 if cfg == 1 else 2e-6
        parity = {"max_rel_l2": float(rel.max()), "median_rel_l2": float(np.median(rel)), "n": int(rel.size),
                  "tol": tol, "pass": bool(rel.max() <= tol),
                  "what": "GPU outputs of the oracle's sampled units of this run vs the fp64 oracle "
                          "(per-unit relative L2; config 9: max relative error of eps, bound, oob)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64" if cfg == 1 else "f32",
                "data": "synthetic",
                "config": {"workload": w["name"], "units_per_gpu": units,
                           "l2": "inputs+outputs exceed the 126 MB L2 (no flush needed)" if cfg != 1 else
                           "tiny (latency-bound), L2-resident",
                           "parallelism": f"dp{world} (independent rows per rank, no collective)"},
                "roofline": roof, "cpu_baseline": cpu, "parity": parity, "quality": quality, "e2e": e2e,
                "gpu_launches": int(launches * args.steps),
                "clocks": clk.summary(),
                "hbm_gbs_algorithmic": achieved}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def quality_numbers(cfg, out, hf, rank):
    """Config 3: relative L2 error of f against the analytic f and of Hf against the 2^20-point
    spectral Hf (BASELINE.json configs[2]) over 16 rows spread over the batch;
    configs 5 / 8: PSNR (peak 255, output clamped to [0, 255], no crop) of the
    distinct benchmarked images against their ground truth."""
    import torch
    c = synth.CONFIGS[cfg]
    if cfg == 3:
        rows = _spread(c["batch"], 16)
        ef, eh = [], []
        for r in rows:
            fr, hr = synth.cfg3_reference(int(r), seed=3 + 1000 * rank)
            ef.append(_rel(out[int(r)].double().cpu().numpy(), fr))
            eh.append(_rel(hf[int(r)].double().cpu().numpy(), hr))
        return {"rows": len(rows), "f_vs_analytic_rel_l2_max": max(ef), "f_vs_analytic_rel_l2_median":
                float(np.median(ef)), "hf_vs_2p20_spectral_rel_l2_max": max(eh),
                "hf_vs_2p20_spectral_rel_l2_median": float(np.median(eh))}
    if cfg in (5, 8):
        if cfg == 5:
            _, truths = synth.cfg5_images(range(4 * rank, 4 * rank + 4))
        else:
            _, truths = synth.sisr_images(range(4 * rank, 4 * rank + 4))
        ps = []
        for i, tr in enumerate(truths):
            o = out[i].double().clamp(0, 255)
            mse = float(((o - torch.from_numpy(np.asarray(tr, dtype=np.float64)).to(o.device)) ** 2).mean())
            ps.append(10 * math.log10(255.0 ** 2 / mse))
        return {"psnr_db": ps, "psnr_db_mean": float(np.mean(ps)), "images": len(ps),
                "what": "PSNR vs the ground-truth image, peak 255, output clamped to [0, 255], no crop"}
    return None


if __name__ == "__main__":
    main()
