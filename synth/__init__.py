"""Seeded synthetic inputs for the MCI hot path (shared by tests, bench and smoke).

This module holds NO arithmetic of the MCI method (no system matrices, no
inverses, no interpolation kernels, no spectrum assembly).  It only *creates
signals* and *samples channel responses* of them, i.e. the forward model the
paper starts from:

  * channel model g_m = f * h_m  <=>  c_m(n) = a(n) b_m(n)
    (convolution theorem, PAPER.md:98-101 Eq. conv and PAPER.md:139-145 Eq. sysfunction);
  * samples at t_n = 2 pi n / N (paper's L is our N);
  * ground truth f(t_p), Hf(t_p) on the output grid.

Both the CUDA path and the oracle consume these inputs; neither is imported
here.  Generators follow SURVEY.md §8(c) items 8-12 and §8(d) "Synthetic
inputs"; the recipes are restated in DESIGN.md §"Input recipe".

Bank description (a Python list, one entry per channel):
    ("identity",)            b(k) = 1
    ("derivative", p)        b(k) = (i k)^p
    ("hilbert",)             b(k) = -i sgn(k)
    ("delay", tau)           b(k) = exp(i k tau)
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "band_indices", "random_band_coeffs", "channel_samples_from_coeffs",
    "grid_from_coeffs", "hilbert_grid_from_coeffs", "phi_coeffs",
    "cfg1", "cfg2_rows", "cfg3_rows", "cfg3_reference", "cfg4_signals",
    "cfg5_images", "image_channels", "bank_of", "CONFIGS",
]

# --------------------------------------------------------------------------
# Channel multipliers of the *forward model* (what the sensor does to f).
# --------------------------------------------------------------------------

def _forward_multiplier(spec, k: np.ndarray) -> np.ndarray:
    """b_m(k) of one channel, vectorised over integer k."""
    kind = spec[0]
    k = np.asarray(k)
    if kind == "identity":
        return np.ones(k.shape, dtype=np.complex128)
    if kind == "derivative":
        return (1j * k.astype(np.float64)) ** int(spec[1])
    if kind == "hilbert":
        return -1j * np.sign(k).astype(np.complex128)
    if kind == "delay":
        return np.exp(1j * k.astype(np.float64) * float(spec[1]))
    raise ValueError(f"unknown channel kind {kind!r}")


def band_indices(M: int, N: int, K1: int | None = None) -> np.ndarray:
    """Integer frequencies of the band I^N = {K1 .. K1+MN-1}.

    Default K1 = -MN/2."""
    MN = M * N
    if K1 is None:
        K1 = -(MN // 2)
    return np.arange(K1, K1 + MN, dtype=np.int64)


def random_band_coeffs(rng: np.random.Generator, MN: int, decay: float | None = None,
                       K1: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Real-signal Fourier coefficients a(k) on the band.

    a(0) ~ N(0,1) real; Re a(k), Im a(k) ~ N(0,1/2) for k>0; a(-k) = conj a(k);
    the unpaired edge a(K1) (when -K1 is out of band) is 0.  Optional decay
    multiplies by 1/(1+|k|/decay).  Draw order: a(0), then (Re, Im) for
    k = 1, 2, ... interleaved.  Returns (k, a)."""
    k = band_indices(1, MN, K1)
    K1 = int(k[0])
    kmax = int(k[-1])
    npos = min(kmax, -K1)  # positive k whose mirror is also in band
    a0 = rng.standard_normal()
    ri = rng.standard_normal(2 * npos) * math.sqrt(0.5)
    apos = ri[0::2] + 1j * ri[1::2]
    a = np.zeros(MN, dtype=np.complex128)
    a[-K1] = a0
    pos = np.arange(1, npos + 1)
    a[pos - K1] = apos
    a[-pos - K1] = np.conj(apos)
    if decay is not None:
        a = a / (1.0 + np.abs(k) / decay)
    return k, a


def channel_samples_from_coeffs(k: np.ndarray, a: np.ndarray, bank, N: int) -> np.ndarray:
    """g_m(t_n) = sum_k a(k) b_m(k) e^{i k t_n}, t_n = 2 pi n/N, n=0..N-1.

    Evaluated by folding the spectrum mod N and one inverse FFT of length N
    (exact sampling of a trigonometric polynomial).  Returns float64 [M][N]
    (real part; the inputs are real signals)."""
    out = np.empty((len(bank), N), dtype=np.float64)
    idx = np.mod(k, N)
    for m, spec in enumerate(bank):
        c = a * _forward_multiplier(spec, k)
        folded = np.zeros(N, dtype=np.complex128)
        np.add.at(folded, idx, c)
        out[m] = np.real(np.fft.ifft(folded) * N)
    return out


def grid_from_coeffs(k: np.ndarray, a: np.ndarray, L: int) -> np.ndarray:
    """Ground truth f(2 pi p/L) = sum_k a(k) e^{2 pi i k p/L} (real part), L >= band width."""
    spec = np.zeros(L, dtype=np.complex128)
    np.add.at(spec, np.mod(k, L), a)
    return np.real(np.fft.ifft(spec) * L)


def hilbert_grid_from_coeffs(k: np.ndarray, a: np.ndarray, L: int) -> np.ndarray:
    """Ground truth Hf(2 pi p/L) with multiplier -i sgn(k)."""
    return grid_from_coeffs(k, a * (-1j * np.sign(k)), L)


# --------------------------------------------------------------------------
# The paper's §5.1 test signal phi.
# --------------------------------------------------------------------------

def phi_coeffs(nmax: int = 600) -> np.ndarray:
    """Taylor coefficients c_n (n=0..nmax) of
        phi(z) = (0.08 z^2 + 0.06 z^10)/((1.3-z)(1.5-z)) + (0.05 z^3 + 0.09 z^10)/((1.2+z)(1.3+z)).
    Uses 1/((a-z)(b-z)) = sum_n z^n (a^{-n-1} - b^{-n-1})/(b-a).  With
    f = Re phi(e^{it}) and Hf = Im phi(e^{it}), the Fourier
    coefficients of f are a(0)=Re c_0, a(n)=c_n/2, a(-n)=conj(c_n)/2."""
    n = np.arange(nmax + 1, dtype=np.float64)

    def base(a, b):
        return (a ** (-(n + 1)) - b ** (-(n + 1))) / (b - a)

    s1 = base(1.3, 1.5)
    s2 = base(-1.2, -1.3)
    c = np.zeros(nmax + 1)

    def add_shift(series, coef, shift):
        c[shift:] += coef * series[: nmax + 1 - shift]

    add_shift(s1, 0.08, 2)
    add_shift(s1, 0.06, 10)
    add_shift(s2, 0.05, 3)
    add_shift(s2, 0.09, 10)
    return c.astype(np.complex128)


# --------------------------------------------------------------------------
# BASELINE.json configs (seeded).  Bank definitions are the configs' own.
# --------------------------------------------------------------------------

CONFIGS = {
    1: dict(M=2, N=32, L=1024, batch=1, bank=[("identity",), ("derivative", 1)], dtype="f64"),
    2: dict(M=3, N=1024, L=16384, batch=65536,
            bank=[("identity",), ("derivative", 1), ("derivative", 2)], dtype="f32"),
    3: dict(M=2, N=4096, L=65536, batch=4096, bank=[("identity",), ("derivative", 1)],
            dtype="f32", hilbert=True),
    4: dict(M=4, N=262144, L=4194304, batch=16,
            bank=[("delay", 2 * math.pi * m / (4 * 262144)) for m in range(4)], dtype="f32"),
    5: dict(Mx=2, My=2, N=512, scale=4, batch=64, size=2048,
            bank=[("identity",), ("derivative", 1)], dtype="f32"),
    # SURVEY.md §8(f) NEXT-1 measurement line: the paper's prime SISR width (PAPER.md:896-931,
    # 321 / 3 = 107) with the (f, f', f'') bank, L = 3N = MN (odd band, odd output length)
    6: dict(M=3, N=107, L=321, batch=65536,
            bank=[("identity",), ("derivative", 1), ("derivative", 2)], dtype="f32"),
    # SURVEY.md §8(f) NEXT-3 measurement line: config-2 rows evaluated at arbitrary points
    7: dict(M=3, N=1024, L=16384, batch=2048, npts=1024,
            bank=[("identity",), ("derivative", 1), ("derivative", 2)], dtype="f32"),
    # SURVEY.md §8(f) NEXT-2 measurement line: the paper's x3 SISR on 510 x 510 images
    # (LR 170 x 170, "Baby (510 x 510)"), 64 synthetic images
    8: dict(H=170, W=170, scale=3, batch=64, dtype="f32"),
    # SURVEY.md §8(f) NEXT-4 measurement line: eps(f, N) of 16,384 spectra on 4x the config-2 band
    9: dict(M=3, N=1024, L=16384, batch=16384, nfreq=4 * 3 * 1024,
            bank=[("identity",), ("derivative", 1), ("derivative", 2)], dtype="f32"),
    # off-benchmark shapes (speed beyond the five benchmark shapes), same
    # generator and about the HBM bytes per step of config 2: two channels (f, f') of N = 2048
    # samples, and four derivative channels (f and its first three derivatives) of N = 1024
    # (MN = 4096 -> L = 16384 = 4 x 4096: the row-kernel family, mci_rowg.cu)
    10: dict(M=2, N=2048, L=16384, batch=65536,
             bank=[("identity",), ("derivative", 1)], dtype="f32"),
    11: dict(M=4, N=1024, L=16384, batch=65536,
             bank=[("identity",), ("derivative", 1), ("derivative", 2), ("derivative", 3)], dtype="f32"),
    # eight time-interleaved channels (tau_m = 2 pi m / (M N): an 8-way interleaved sampler,
    # PAPER.md:139-147 with delay systems) of N = 512 samples -> L = 16384
    12: dict(M=8, N=512, L=16384, batch=65536,
             bank=[("delay", 2 * math.pi * m / (8 * 512)) for m in range(8)], dtype="f32"),
}


def error_spectra(batch: int, k_lo: int, nfreq: int, seed: int = 9, block: int = 1024) -> np.ndarray:
    """Config 9 inputs: complex64 spectra a(k), k = k_lo .. k_lo + nfreq - 1, Re/Im ~ N(0, 1/2)
    scaled by 1/(1+|k|/256) (the config-2 decay extended beyond the band); rows drawn in blocks
    of `block` from default_rng([seed, block index])."""
    k = np.arange(k_lo, k_lo + nfreq)
    sc = (1.0 / (1.0 + np.abs(k) / 256.0)).astype(np.float32)
    out = np.empty((batch, nfreq), dtype=np.complex64)
    for b0 in range(0, batch, block):
        nb = min(block, batch - b0)
        rng = np.random.default_rng([seed, b0 // block])
        z = rng.standard_normal((nb, 2 * nfreq), dtype=np.float32) * np.float32(math.sqrt(0.5))
        out[b0:b0 + nb] = (z[:, 0::2] + 1j * z[:, 1::2]) * sc
    return out


def offgrid_points(npts: int, seed: int = 7) -> np.ndarray:
    """Evaluation points for config 7: uniform in [0, 2 pi), seeded (float64)."""
    return np.random.default_rng([seed, 777]).uniform(0.0, 2 * math.pi, npts)


def bank_of(cfg: int):
    return CONFIGS[cfg]["bank"]


def cfg1(seed: int = 0):
    """Config 1: one real trig polynomial, MN=64 (k=-32..31), bank (1, ik), N=32, L=1024, fp64."""
    c = CONFIGS[1]
    rng = np.random.default_rng(seed)
    k, a = random_band_coeffs(rng, c["M"] * c["N"])
    g = channel_samples_from_coeffs(k, a, c["bank"], c["N"])[None]
    return dict(g=g, k=k, a=a[None], truth=grid_from_coeffs(k, a, c["L"])[None])


_CFG2_BLOCK = 256


def cfg2_rows(rows, seed: int = 2, with_truth: bool = False, M=None, N=None, L=None, bank=None):
    """Config 2 rows (by global row index): random trig polynomials, MN=3072,
    a(k) scaled by 1/(1+|k|/256), bank (1, ik, -k^2), N=1024.

    Row r's coefficients come from default_rng([seed, r // 256]) drawing 256
    rows in order, so any subset is reproducible.  Returns float32 g[R][M][N]
    (cast from fp64) and optionally fp64 truth on L points."""
    c = CONFIGS[2]
    M = M or c["M"]; N = N or c["N"]; L = L or c["L"]; bank = bank or c["bank"]
    rows = np.asarray(rows, dtype=np.int64)
    MN = M * N
    g = np.empty((len(rows), M, N), dtype=np.float32)
    truth = np.empty((len(rows), L), dtype=np.float64) if with_truth else None
    cache: dict[int, list] = {}
    for i, r in enumerate(rows):
        blk = int(r) // _CFG2_BLOCK
        if blk not in cache:
            rng = np.random.default_rng([seed, blk])
            cache = {blk: [random_band_coeffs(rng, MN, decay=256.0) for _ in range(_CFG2_BLOCK)]}
        k, a = cache[blk][int(r) % _CFG2_BLOCK]
        g[i] = channel_samples_from_coeffs(k, a, bank, N)
        if with_truth:
            truth[i] = grid_from_coeffs(k, a, L)
    return (g, truth) if with_truth else g


def cfg2_batch_fast(batch: int, seed: int = 2, M=3, N=1024, bank=None):
    """Vectorised generator for the full config-2 batch (bench/large parity).

    Same distribution as cfg2_rows but drawn per 256-row block in one shot;
    rows are identical to cfg2_rows(r) (same generator, same draw order)."""
    bank = bank or CONFIGS[2]["bank"]
    MN = M * N
    out = np.empty((batch, M, N), dtype=np.float32)
    K1 = -(MN // 2)
    k = np.arange(K1, K1 + MN)
    npos = min(K1 + MN - 1, -K1)  # same as random_band_coeffs
    mult = np.stack([_forward_multiplier(s, k) for s in bank])  # [M][MN]
    scale = 1.0 / (1.0 + np.abs(k) / 256.0)
    idx = np.mod(k, N)
    for b0 in range(0, batch, _CFG2_BLOCK):
        nb = min(_CFG2_BLOCK, batch - b0)
        rng = np.random.default_rng([seed, b0 // _CFG2_BLOCK])
        A = np.zeros((_CFG2_BLOCK, MN), dtype=np.complex128)
        for i in range(_CFG2_BLOCK):
            a0 = rng.standard_normal()
            ri = rng.standard_normal(2 * npos) * math.sqrt(0.5)
            ap = ri[0::2] + 1j * ri[1::2]
            A[i, -K1] = a0
            A[i, 1 - K1: npos + 1 - K1] = ap
            A[i, -K1 - npos: -K1][::-1] = np.conj(ap)
        A = A[:nb] * scale
        for m in range(M):
            c = A * mult[m]
            # fold mod N: the band is M*N consecutive k starting at K1
            folded = np.roll(c.reshape(nb, MN // N, N).sum(axis=1), int(idx[0]), axis=1)
            out[b0:b0 + nb, m] = np.real(np.fft.ifft(folded, axis=1) * N)
    return out


# ---- config 3: non-bandlimited bumps + smoothed periodic step --------------

def _cfg3_params(rng):
    A = rng.standard_normal(8)
    c = rng.uniform(0.0, 2 * math.pi, 8)
    w = rng.uniform(0.02, 0.3, 8)
    As = rng.standard_normal()
    cs = rng.uniform(0.0, 2 * math.pi)
    return A, c, w, As, cs


def _cfg3_eval(params, t):
    """f(t) and f'(t) (analytic) for the config-3 signal."""
    A, c, w, As, cs = params
    f = np.zeros_like(t)
    fp = np.zeros_like(t)
    for i in range(8):
        for j in (-1, 0, 1):
            d = t - c[i] + 2 * math.pi * j
            e = np.exp(-d * d / (2 * w[i] ** 2))
            f += A[i] * e
            fp += A[i] * e * (-d / w[i] ** 2)
    x = np.sin(t - cs) / 0.01
    s = 0.5 * (1.0 + np.tanh(0.5 * x))  # logistic, overflow-free
    f += As * s
    fp += As * s * (1.0 - s) * np.cos(t - cs) / 0.01
    return f, fp


def cfg3_rows(rows, seed: int = 3, N: int = 4096):
    """Config 3 channel samples (f, f') at t_n = 2 pi n/N, float32 [R][2][N]."""
    rows = np.asarray(rows, dtype=np.int64)
    g = np.empty((len(rows), 2, N), dtype=np.float32)
    t = 2 * math.pi * np.arange(N) / N
    for i, r in enumerate(rows):
        p = _cfg3_params(np.random.default_rng([seed, int(r)]))
        f, fp = _cfg3_eval(p, t)
        g[i, 0] = f
        g[i, 1] = fp
    return g


def cfg3_reference(row: int, L: int = 65536, seed: int = 3, nref: int = 1 << 20):
    """Analytic f on L points and Hf from a 2^20-point spectral reference
    (BASELINE.json config 3), subsampled to L points."""
    p = _cfg3_params(np.random.default_rng([seed, int(row)]))
    t = 2 * math.pi * np.arange(nref) / nref
    f, _ = _cfg3_eval(p, t)
    F = np.fft.fft(f)
    kk = np.fft.fftfreq(nref, d=1.0 / nref)
    hf = np.real(np.fft.ifft(-1j * np.sign(kk) * F))
    step = nref // L
    return f[::step].copy(), hf[::step].copy()


# ---- config 4: long delay-bank signals -------------------------------------

def cfg4_signals(signals, seed: int = 4, M: int = 4, N: int = 262144):
    """Config 4: real trig polynomials with MN coefficients (cfg2 distribution),
    sampled through the delay bank tau_m = 2 pi m/(MN): g_m(t_n) = f(t_n + tau_m)
    = the interleaved uniform samples x[M n + m].
    Returns (g float32 [S][M][N], coefficient list)."""
    signals = np.asarray(signals, dtype=np.int64)
    MN = M * N
    g = np.empty((len(signals), M, N), dtype=np.float32)
    coeffs = []
    for i, s in enumerate(signals):
        rng = np.random.default_rng([seed, int(s)])
        k, a = random_band_coeffs(rng, MN, decay=256.0)
        x = grid_from_coeffs(k, a, MN)  # uniform samples at 2 pi u/(MN)
        g[i] = x.reshape(N, M).T
        coeffs.append((k, a))
    return g, coeffs


# ---- config 5: SISR-shaped 2D images ----------------------------------------

def cfg5_image(index: int, seed: int = 5, size: int = 2048, corr: float = 16.0, shapes: int = 20):
    """Ground-truth image: GRF (white noise filtered by
    exp(-|k|^2 l^2/2), l = corr px, mean 128, std 40) plus `shapes` filled
    rectangles/disks with random intensities, wrapped periodically; clipped to
    [0,255], rounded to uint8, returned as float64."""
    rng = np.random.default_rng([seed, int(index)])
    w = rng.standard_normal((size, size))
    kx = 2 * math.pi * np.fft.fftfreq(size)
    ky = 2 * math.pi * np.fft.rfftfreq(size)
    filt = np.exp(-(kx[:, None] ** 2 + ky[None, :] ** 2) * corr * corr / 2)
    grf = np.fft.irfft2(np.fft.rfft2(w) * filt, s=(size, size))
    grf = 128.0 + 40.0 * (grf - grf.mean()) / grf.std()
    img = grf
    yy = np.arange(size)[:, None]
    xx = np.arange(size)[None, :]
    for _ in range(shapes):
        kind = rng.integers(0, 2)
        cy, cx = rng.uniform(0, size, 2)
        val = rng.uniform(0, 255)
        dy = (yy - cy + size / 2) % size - size / 2  # periodic wrap
        dx = (xx - cx + size / 2) % size - size / 2
        if kind == 0:
            hh, hw = rng.uniform(size / 64, size / 8, 2)
            mask = (np.abs(dy) <= hh) & (np.abs(dx) <= hw)
        else:
            rad = rng.uniform(size / 64, size / 10)
            mask = dy * dy + dx * dx <= rad * rad
        img = np.where(mask, val, img)
    return np.round(np.clip(img, 0, 255)).astype(np.uint8).astype(np.float64)


def image_channels(img: np.ndarray, N: int, bank=None) -> np.ndarray:
    """Channel images of the tensor bank {b_x} (x) {b_y} decimated to N x N
    (SURVEY.md §8(c) item 11): the image is one period of a 2D trig polynomial,
    derivatives are w.r.t. t in [0, 2 pi) (integer wavenumbers), Nyquist mode
    zeroed for odd derivatives.  Layout [My][Mx][N][N] = [my][mx][ny][nx]."""
    bank = bank or CONFIGS[5]["bank"]
    size = img.shape[0]
    step = size // N
    F = np.fft.fft2(img)
    kk = np.fft.fftfreq(size, d=1.0 / size)
    nyq = np.abs(kk) == size // 2
    out = np.empty((len(bank), len(bank), N, N), dtype=np.float64)
    for my, sy in enumerate(bank):
        by = _forward_multiplier(sy, kk.astype(np.int64))
        if sy[0] == "derivative" and int(sy[1]) % 2 == 1:
            by = np.where(nyq, 0, by)
        for mx, sx in enumerate(bank):
            bx = _forward_multiplier(sx, kk.astype(np.int64))
            if sx[0] == "derivative" and int(sx[1]) % 2 == 1:
                bx = np.where(nyq, 0, bx)
            ch = np.real(np.fft.ifft2(F * by[:, None] * bx[None, :]))
            out[my, mx] = ch[::step, ::step]
    return out


def cfg5_images(indices, seed: int = 5, size: int = 2048, N: int = 512):
    """Config 5 inputs: float32 channels [I][My][Mx][N][N] and float64 ground truths."""
    indices = list(indices)
    g = np.empty((len(indices), 2, 2, N, N), dtype=np.float32)
    truths = []
    for i, ix in enumerate(indices):
        img = cfg5_image(ix, seed=seed, size=size)
        g[i] = image_channels(img, N)
        truths.append(img)
    return g, truths


# ---- SISR inputs -----------------------------
def gaussian_blur_5x5(img: np.ndarray, sigma: float = 1.0) -> np.ndarray:
    """5 x 5 Gaussian blur, standard deviation sigma, normalised, periodic boundary
    (the paper's step 1; periodic to match the periodic signal model)."""
    ax = np.arange(-2, 3)
    k1 = np.exp(-ax * ax / (2.0 * sigma * sigma))
    k1 /= k1.sum()
    out = np.zeros_like(img, dtype=np.float64)
    for dy in range(5):
        for dx in range(5):
            out += k1[dy] * k1[dx] * np.roll(np.roll(img, ax[dy], axis=0), ax[dx], axis=1)
    return out


def sisr_images(indices, hr_size: int = 510, scale: int = 3, seed: int = 8):
    """SISR workload: HR ground truths (the config-5 generator at hr_size, periodic),
    blurred 5x5 / sigma 1 and decimated by `scale` at phase 0 -> LR float32 [I][H][W]."""
    indices = list(indices)
    n = hr_size // scale
    lr = np.empty((len(indices), n, n), dtype=np.float32)
    hrs = []
    for i, ix in enumerate(indices):
        hr = cfg5_image(ix, seed=seed, size=hr_size, corr=4.0, shapes=12)
        lr[i] = gaussian_blur_5x5(hr)[::scale, ::scale]
        hrs.append(hr)
    return lr, hrs
