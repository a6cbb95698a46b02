"""Seeded generators: determinism, subset reproducibility, declared shapes."""
import math

import numpy as np

import synth


def test_cfg2_fast_equals_rows():
    fast = synth.cfg2_batch_fast(600)
    rows = [0, 1, 255, 256, 599]
    ref = synth.cfg2_rows(rows)
    assert np.array_equal(fast[rows], ref)
    assert fast.dtype == np.float32 and fast.shape == (600, 3, 1024)


def test_cfg2_rows_truth_bandlimited():
    g, truth = synth.cfg2_rows([3], with_truth=True)
    # identity channel = truth at the coarse sites t_n (L/N = 16)
    assert np.max(np.abs(g[0, 0] - truth[0, ::16])) < 1e-5 * np.max(np.abs(truth))


def test_cfg3_deterministic_and_derivative():
    a = synth.cfg3_rows([7], N=1024)
    b = synth.cfg3_rows([7], N=1024)
    assert np.array_equal(a, b)
    # analytic derivative vs spectral derivative of the sampled signal
    g = synth.cfg3_rows([7], N=4096)[0].astype(np.float64)
    F = np.fft.fft(g[0])
    k = np.fft.fftfreq(4096, d=1 / 4096)
    spec = np.real(np.fft.ifft(1j * k * F))
    assert np.max(np.abs(spec - g[1])) < 1e-2 * np.max(np.abs(g[1]))


def test_cfg4_interleaving():
    g, coeffs = synth.cfg4_signals([0], M=4, N=64)
    k, a = coeffs[0]
    t = 2 * math.pi * np.arange(64) / 64
    for m in range(4):
        tau = 2 * math.pi * m / 256
        ref = np.real(np.exp(1j * np.outer(t + tau, k)) @ a)
        assert np.max(np.abs(g[0, m] - ref)) < 1e-5 * np.max(np.abs(ref))


def test_cfg5_image_small():
    img = synth.cfg5_image(0, size=128, corr=4.0, shapes=3)
    assert img.shape == (128, 128) and img.min() >= 0 and img.max() <= 255
    assert np.all(img == np.round(img))
    ch = synth.image_channels(img, 32)
    assert ch.shape == (2, 2, 32, 32)
    assert np.array_equal(ch[0, 0], img[::4, ::4]) or np.max(np.abs(ch[0, 0] - img[::4, ::4])) < 1e-9
