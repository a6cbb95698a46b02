"""Every kernel and variant of libmci.so at reduced sizes, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/sanitize.sh runs this script under each tool).

Inputs are seeded random channel data; the results are not checked here (the parity
tests do that), only that every launch completes without a sanitizer report.  Each case
names the kernel(s) it drives and the environment switch that selects the variant."""
from __future__ import annotations

import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_10291_b200 as mci  # noqa: E402

F, FD, FDD = [("identity",)], [("identity",), ("derivative", 1)], [("identity",), ("derivative", 1), ("derivative", 2)]
rng = np.random.default_rng(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rnd(*shape, dtype=np.float32):
    return rng.standard_normal(shape).astype(dtype)


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        fn()
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def row_kernel():  # mci_row_kernel, every MCI_ROW_VARIANT, closed form and Q~ table
    g = dev(rnd(5, 3, 1024))
    for v in ["0", "1", "2", "3", "4", "5", "6", "7", "8"]:
        for q in ["0", "1"]:
            with_env({"MCI_ROW_VARIANT": v, "MCI_ROW_QTAB": q}, lambda: mci.Plan(3, 1024, 16384, FDD).execute(g))


def hilbert_kernel():  # mci_hilbert_kernel (store warpgroup / direct stores)
    g = dev(rnd(3, 2, 4096))
    for v in ["0", "1"]:
        with_env({"MCI_HILBERT_VARIANT": v}, lambda: mci.Plan(2, 4096, 65536, FD, hilbert=True).execute(g))


def fused_kernel():  # mci_fused_kernel (generic power-of-two), fp32/fp64, real and analytic
    for dt, npdt in (("f32", np.float32), ("f64", np.float64)):
        g = dev(rnd(7, 2, 64, dtype=npdt))
        mci.Plan(2, 64, 1024, FD, dtype=dt).execute(g)
        mci.Plan(2, 64, 1024, FD, dtype=dt, hilbert=True).execute(g)
    with_env({"MCI_DISABLE_ROW": "1"}, lambda: mci.Plan(3, 1024, 16384, FDD).execute(dev(rnd(3, 3, 1024))))


def line_kernel():  # mci_line_kernel: 1D contiguous (prefetch / direct), 2D passes and their variants
    g = dev(rnd(40, 2, 512))
    for pf in ["1", "0"]:
        for lv in ["0", "1"]:
            with_env({"MCI_LINE_PF": pf, "MCI_LINE_VARIANT": lv}, lambda: mci.Plan(2, 512, 2048, FD).execute(g))
    gi = dev(rnd(2, 2, 2, 512, 512))
    envs = [{}, {"MCI_LINE_TMA": "0"}, {"MCI_LINE_G16": "0"}, {"MCI_LINE_CT8": "1"}, {"MCI_2D_TSTORE": "0"},
            {"MCI_2D_ORDER": "1"}, {"MCI_LINE_VARIANT": "1"}, {"MCI_2D_STREAMS": "2", "MCI_2D_WS_MB": "24"}]
    for e in envs:
        with_env(e, lambda: mci.Plan2D(2, 512, FD, 2, 512, FD, 4).execute(gi))


def fourstep():  # mci_fs_max + mci_fsf_fa/fb/ic (fast, delay bank) and the generic four-step kernels
    M, N = 4, 262144
    bank = [("delay", 2 * math.pi * m / (M * N)) for m in range(M)]
    g = dev(rnd(2, M, N))
    with_env({"MCI_FS_WS_MB": "64"}, lambda: mci.Plan(M, N, 4 * M * N, bank).execute(g))
    with_env({"MCI_FOURSTEP_GENERIC": "1"}, lambda: mci.Plan(M, N, 4 * M * N, bank).execute(g))
    g2 = dev(rnd(2, 2, 16384))
    mci.Plan(2, 16384, 131072, FD).execute(g2)


def anylen():  # mci_anylen_kernel: mixed radix, Bluestein (prime 107), odd band, analytic, fp64
    g = dev(rnd(9, 3, 107))
    mci.Plan(3, 107, 321, FDD).execute(g)
    mci.Plan(3, 107, 321, FDD, hilbert=True).execute(g)
    mci.Plan(3, 107, 321, FDD, dtype="f64").execute(dev(rnd(9, 3, 107, dtype=np.float64)))
    mci.Plan(2, 170, 510, FD).execute(dev(rnd(5, 2, 170)))
    with_env({"MCI_FORCE_ANYLEN": "1"}, lambda: mci.Plan(2, 64, 256, FD).execute(dev(rnd(5, 2, 64))))
    mci.Plan2D(2, 60, FD, 2, 56, FD, 3).execute(dev(rnd(2, 2, 2, 56, 60)))


def offgrid_complex_analysis():  # off-grid Horner, complex output, residual, averaged error
    p = mci.Plan(3, 107, 321, FDD, offgrid=True)
    p.execute_offgrid(dev(rnd(4, 3, 107)), dev(rng.uniform(0, 2 * np.pi, 33).astype(np.float32)))
    pc = mci.Plan(2, 64, 256, [("delay", 0.0), ("delay", 0.01)], complex=True, K1=-10)
    gc = (rnd(3, 2, 64) + 1j * rnd(3, 2, 64)).astype(np.complex64)
    pc.execute(dev(gc))
    pa = mci.Plan(2, 64, 256, FD, analysis=True)
    pa.consistency_residual(dev(rnd(5, 2, 64)))
    spec = (rnd(6, 300) + 1j * rnd(6, 300)).astype(np.complex64)
    pa.averaged_error(dev(spec), -150)


def sisr():  # mci_sisr_fd_rows/cols + anylen passes + transpose
    mci.SisrPlan(14, 18, 3).execute(dev(rnd(2, 14, 18)))
    mci.SisrPlan(20, 20, 4, dtype="f64").execute(dev(rnd(1, 20, 20, dtype=np.float64)))


CASES = [row_kernel, hilbert_kernel, fused_kernel, line_kernel, fourstep, anylen, offgrid_complex_analysis, sisr]

if __name__ == "__main__":
    want = sys.argv[1:]
    for c in CASES:
        if want and c.__name__ not in want:
            continue
        c()
        torch.cuda.synchronize()
        print(f"case {c.__name__} done", flush=True)
