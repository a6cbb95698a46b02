"""Pins of the fp64 oracle against things other than itself.

Every expected value here comes from the paper (printed numbers / closed
forms, cited), from textbook identities, from brute-force dense solves
(numpy.linalg), or from ground-truth synthesis -- never from the oracle's own
code path and never from the CUDA path.
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def bmult(spec, k):
    """Channel multipliers retyped from the paper, independent of oracle and synth."""
    k = np.asarray(k, dtype=np.float64)
    if spec[0] == "identity":
        return np.ones_like(k, dtype=complex)
    if spec[0] == "derivative":
        return (1j * k) ** spec[1]
    if spec[0] == "hilbert":
        return -1j * np.sign(k)
    if spec[0] == "delay":
        return np.exp(1j * k * spec[1])
    raise ValueError(spec)


BANKS = {
    "identity": [("identity",)],
    "f_df": [("identity",), ("derivative", 1)],
    "f_df_ddf": [("identity",), ("derivative", 1), ("derivative", 2)],
    "f_hf": [("identity",), ("hilbert",)],
    "delay4": "delay",
}


def bank_for(name, N):
    if name == "delay4":
        return [("delay", 2 * math.pi * m / (4 * N)) for m in range(4)]
    return BANKS[name]


# ---------------------------------------------------------------- P1 ------------
@pytest.mark.parametrize("name,N,L", [("identity", 64, 256), ("f_df", 32, 512), ("f_df_ddf", 16, 192),
                                      ("f_hf", 16, 256), ("delay4", 8, 128), ("f_df", 8, 16)])
def test_p1_exact_reconstruction(name, N, L):
    """Theorem 1: f in B_N is reproduced exactly, and so is Hf
    (Example 6). Expected = closed form sum a(k) e^{ikt}."""
    bank = bank_for(name, N)
    M = len(bank)
    rng = np.random.default_rng(11)
    k, a = synth.random_band_coeffs(rng, M * N)
    g = synth.channel_samples_from_coeffs(k, a, bank, N)
    P = oracle.OraclePlan(M, N, L, bank)
    t = 2 * np.pi * np.arange(L) / L
    closed = np.real(np.exp(1j * np.outer(t, k)) @ a)
    closed_h = np.real(np.exp(1j * np.outer(t, k)) @ (a * -1j * np.sign(k)))
    assert rel(P.eval(g[None])[0], closed) < 1e-12
    assert rel(P.eval(g[None], hilbert=True)[0], closed_h) < 1e-12


# ---------------------------------------------------------------- P2 ------------
def test_p2_dirichlet_odd_band():
    """Example 1: M = 1, band -n0..n0 => y = D_{n0}, the Dirichlet
    kernel sin((n0+1/2)t)/sin(t/2), value 2 n0 + 1 at t = 0."""
    n0 = 7
    N = 2 * n0 + 1
    L = 4 * N
    P = oracle.OraclePlan(1, N, L, [("identity",)], K1=-n0)
    Y = P.kernel_table()[0]
    t = 2 * np.pi * np.arange(L) / L
    with np.errstate(divide="ignore", invalid="ignore"):
        D = np.sin((n0 + 0.5) * t) / np.sin(t / 2)
    D[0] = 2 * n0 + 1
    assert np.max(np.abs(Y - D)) < 1e-12 * N


def test_p2_dirichlet_even_band():
    """Even band -K..K-1: y(t) = sum e^{ikt} = e^{-it/2} sin(Kt)/sin(t/2) (geometric sum)."""
    K = 16
    N = 2 * K
    L = 8 * N
    P = oracle.OraclePlan(1, N, L, [("identity",)])
    Y = P.kernel_table()[0]
    t = 2 * np.pi * np.arange(L) / L
    with np.errstate(divide="ignore", invalid="ignore"):
        D = np.cos(t / 2) * np.sin(K * t) / np.sin(t / 2)
    D[0] = 2 * K
    assert np.max(np.abs(Y - D)) < 1e-12 * N


# ---------------------------------------------------------------- P3 ------------
@pytest.mark.parametrize("name,N,L", [("f_df", 8, 64), ("f_df_ddf", 8, 96), ("f_hf", 12, 96),
                                      ("delay4", 4, 64), ("identity", 24, 96), ("f_df_ddf", 5, 60)])
def test_p3_dense_solve_any_data(name, N, L):
    """Arbitrary real channel data (not band-limited): T_N f is the unique in-band
    trig polynomial whose channel samples equal g (consistency + uniqueness,
    PAPER.md:302-305, 546-585).  Brute force: one dense MN x MN complex solve."""
    bank = bank_for(name, N)
    M = len(bank)
    MN = M * N
    rng = np.random.default_rng(5)
    g = rng.standard_normal((M, N))
    k = np.arange(-(MN // 2), -(MN // 2) + MN)
    n = np.arange(N)
    A = np.concatenate([bmult(b, k)[None, :] * np.exp(2j * np.pi * np.outer(n, k) / N) for b in bank])
    a = np.linalg.solve(A, g.reshape(-1).astype(complex))
    t = 2 * np.pi * np.arange(L) / L
    E = np.exp(1j * np.outer(t, k))
    P = oracle.OraclePlan(M, N, L, bank)
    assert rel(P.eval(g[None])[0], np.real(E @ a)) < 1e-11
    assert rel(P.eval(g[None], hilbert=True)[0], np.real(E @ (a * -1j * np.sign(k)))) < 1e-11
    # off-grid definition path agrees with the grid path
    assert rel(P.eval_offgrid(g, t), np.real(E @ a)) < 1e-11


# ---------------------------------------------------------------- P4 ------------
def test_p4_example2_inverse_and_kernels():
    """Example 2, bank (f, f', f''), band -N'..N' with
    N' = 3 N0 + 1 and (paper) L = 2 N0 + 1 = our N: printed H_n^{-1} and the
    closed forms of y_1, y_2, y_3."""
    N0 = 3
    Lp = 2 * N0 + 1              # paper's L = samples per channel = our N
    Np = 3 * N0 + 1              # paper's N (band half-width)
    bank = BANKS["f_df_ddf"]
    Lout = 8 * Lp
    P = oracle.OraclePlan(3, Lp, Lout, bank, K1=-Np)
    for jj in range(Lp):
        n = -Np + jj
        L = float(Lp)
        printed = np.array([
            [(2 * L**2 + 3 * L * n + n**2) / (2 * L**2), -n * (2 * L + n) / L**2, n * (L + n) / (2 * L**2)],
            [1j * (3 * L + 2 * n) / (2 * L**2), -2j * (L + n) / L**2, 1j * (L + 2 * n) / (2 * L**2)],
            [-1 / (2 * L**2), 1 / L**2, -1 / (2 * L**2)],
        ])
        assert np.max(np.abs(P.Q[jj] - printed)) < 1e-13
    s = np.arange(1, Lout)
    t = 2 * np.pi * s / Lout
    c3 = np.sin((N0 + 0.5) * t) ** 3
    den = (2 * N0 + 1) ** 2
    y1 = c3 * (N0**2 + N0 + 1 - (N0 + 1) * N0 * np.cos(t)) / (den * np.sin(t / 2) ** 3)
    y2 = np.sin(t) * c3 / (den * np.sin(t / 2) ** 3)
    y3 = 2 * c3 / (den * np.sin(t / 2))
    kk = np.arange(-Np, Np + 1)
    for m, y in enumerate((y1, y2, y3)):
        full = np.exp(1j * np.outer(t, kk)) @ P.r[m]   # complex y_m from the oracle's r_m
        assert np.max(np.abs(full - y)) < 1e-12 * Lp
        assert np.max(np.abs(P.kernel_table()[m][1:] - y)) < 1e-12 * Lp


# ---------------------------------------------------------------- P5 ------------
def _table_rows():
    rows = []
    with open(os.path.join(HERE, "golden", "table_approximated.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                p = line.split()
                rows.append(tuple(int(x) for x in p[:5]) + (float(p[5]), float(p[6])))
    return rows


def _half_unit_4sig(x):
    e = math.floor(math.log10(abs(x)))
    return 0.5 * 10 ** (e - 3)


@pytest.mark.parametrize("row", _table_rows(), ids=lambda r: f"mu{r[0]}_f{r[1]}_hf{r[2]}_d{r[3]}")
def test_p5_paper_table(row):
    """Table approximatedtable: delta1/delta2 of T_N on phi.
    Readings: band K1 = -mu/2, output Re T_N f, delta2 = ||Hf - H(Re T_N f)||/||Hf||
    (SURVEY.md §8(c) items 2, 3, 5).  31 of 32 printed values must match to the
    printed 4 significant digits; the mu=96 (48 f + 48 Hf) delta2 is a likely
    misprint (reading R9) and is held to 1 %."""
    mu, nf, nh, n1, n2, d1, d2 = row
    c = synth.phi_coeffs(600)
    j = np.arange(len(c))

    def ev(t, mult):
        return np.exp(1j * np.outer(t, j)) @ (c * mult)

    if nh:
        bank, N = BANKS["f_hf"], nf
    elif n1:
        bank, N = BANKS["f_df_ddf"], nf
    else:
        bank, N = BANKS["identity"], nf
    tn = 2 * np.pi * np.arange(N) / N
    g = []
    for b in bank:
        if b[0] == "identity":
            g.append(np.real(ev(tn, 1)))
        elif b[0] == "hilbert":
            g.append(np.imag(ev(tn, 1)))
        else:
            g.append(np.real(ev(tn, (1j * j) ** b[1])))
    tp = 2 * np.pi * np.arange(2048) / 2048
    f_true, hf_true = np.real(ev(tp, 1)), np.imag(ev(tp, 1))
    P = oracle.OraclePlan(len(bank), N, 2048, bank)
    e1 = rel(P.eval_offgrid(np.array(g), tp), f_true)
    e2 = rel(P.eval_offgrid(np.array(g), tp, hilbert=True), hf_true)
    assert abs(e1 - d1) <= 1.05 * _half_unit_4sig(d1)
    if (mu, nh) == (96, 48):
        assert abs(e2 / d2 - 1) < 0.01       # printed 0.3836e-2, computed 0.3869e-2
    else:
        assert abs(e2 - d2) <= 1.05 * _half_unit_4sig(d2)


# ---------------------------------------------------------------- P6 ------------
@pytest.mark.parametrize("name,N,L", [("f_df", 16, 256), ("f_df_ddf", 8, 96), ("f_hf", 8, 64), ("identity", 32, 128)])
def test_p6_consistency_identity_channel(name, N, L):
    """Consistency theorem for any finite-energy f: T_N f
    reproduces the samples of the identity channel at t_n."""
    bank = bank_for(name, N)
    M = len(bank)
    g = np.random.default_rng(3).standard_normal((M, N))
    out = oracle.OraclePlan(M, N, L, bank).eval(g[None])[0]
    assert np.max(np.abs(out[:: L // N] - g[0])) < 1e-12 * np.max(np.abs(g)) * M


def test_p6_consistency_delay_bank():
    """Delay bank: output at p = (L/N) n + (L/MN) m equals g_m[n] (t_n + tau_m)."""
    M, N, L = 4, 16, 256
    bank = bank_for("delay4", N)
    g = np.random.default_rng(4).standard_normal((M, N))
    out = oracle.OraclePlan(M, N, L, bank).eval(g[None])[0]
    for m in range(M):
        assert np.max(np.abs(out[m * (L // (M * N)):: L // N] - g[m])) < 1e-12 * 10


# ---------------------------------------------------------------- P7 ------------
@pytest.mark.parametrize("name,N", [("f_df", 16), ("f_df_ddf", 12), ("f_hf", 10), ("delay4", 6)])
def test_p7_biorthogonality(name, N):
    """Lemma rmbm: sum_m r_m(n) b_m(n) = 1 on the band and
    sum_m r_m(n1) b_m(n2) = 0 when (n1 - n2)/N is a nonzero integer."""
    bank = bank_for(name, N)
    M = len(bank)
    P = oracle.OraclePlan(M, N, 4 * M * N, bank)
    k = np.arange(P.K1, P.K1 + M * N)
    B = np.array([bmult(b, k) for b in bank])              # B[m][k]
    S = P.r.T @ B                                          # S[k1][k2] = sum_m r_m(k1) b_m(k2)
    for i in range(M * N):
        assert abs(S[i, i] - 1) < 1e-12
        for l in range(M):
            j2 = (i % N) + l * N
            if j2 != i:
                assert abs(S[i, j2]) < 1e-12 * max(1.0, np.max(np.abs(B)))


# ---------------------------------------------------------------- P8 ------------
def test_p8_hilbert_pairs_and_antiinvolution():
    """H{cos kt} = sin kt, H{sin kt} = -cos kt and
    H^2 f = -f + a(0) (Eq. Hsquare)."""
    M, N, L = 2, 16, 128
    bank = BANKS["f_df"]
    tn = 2 * np.pi * np.arange(N) / N
    tp = 2 * np.pi * np.arange(L) / L
    f = lambda t: 0.7 + np.cos(3 * t) + 0.5 * np.sin(5 * t)
    df = lambda t: -3 * np.sin(3 * t) + 2.5 * np.cos(5 * t)
    P = oracle.OraclePlan(M, N, L, bank)
    hf = P.eval(np.array([f(tn), df(tn)])[None], hilbert=True)[0]
    hf_true = np.sin(3 * tp) - 0.5 * np.cos(5 * tp)
    assert np.max(np.abs(hf - hf_true)) < 1e-12
    # apply H again: feed samples of Hf (and its derivative) back
    dhf = lambda t: 3 * np.cos(3 * t) + 2.5 * np.sin(5 * t)
    h2 = P.eval(np.array([np.sin(3 * tn) - 0.5 * np.cos(5 * tn), dhf(tn)])[None], hilbert=True)[0]
    assert np.max(np.abs(h2 - (-f(tp) + 0.7))) < 1e-12


def test_p8_discrete_analytic_signal_one_sided():
    """Remark after Example 3: the DFT of out + i Hout has no
    negative-frequency content (Z(k) = X(0), 2X(k), 0)."""
    M, N, L = 3, 16, 192
    bank = BANKS["f_df_ddf"]
    g = np.random.default_rng(8).standard_normal((M, N))
    P = oracle.OraclePlan(M, N, L, bank)
    z = P.eval(g[None])[0] + 1j * P.eval(g[None], hilbert=True)[0]
    Z = np.fft.fft(z)
    X = np.fft.fft(P.eval(g[None])[0])
    assert np.max(np.abs(Z[L // 2 + 1:])) < 1e-11 * np.max(np.abs(Z))
    assert np.max(np.abs(Z[1:L // 2] - 2 * X[1:L // 2])) < 1e-11 * np.max(np.abs(Z))


# ---------------------------------------------------------------- P9 ------------
def test_p9_delay_closed_form_and_textbook_interpolation():
    """Delay bank = interlaced uniform sampling: (a) closed-form kernel equals the
    generic kernel table; (b) closed-form point evaluation equals grid
    evaluation; (c) both equal textbook FFT trig interpolation of the
    interleaved MN-point sequence (real part, band -K..K-1)."""
    M, N, L = 4, 8, 128
    bank = bank_for("delay4", N)
    P = oracle.OraclePlan(M, N, L, bank)
    assert np.max(np.abs(oracle.delay_kernel_table(M, N, L) - P.kernel_table())) < 1e-12 * M * N
    g = np.random.default_rng(9).standard_normal((M, N))
    grid = P.eval(g[None])[0]
    pts = np.array([0, 1, 5, 17, 63, 64, 127])
    assert np.max(np.abs(oracle.delay_eval_points(M, N, L, g, pts) - grid[pts])) < 1e-12
    x = g.T.reshape(-1)                                   # x[M n + m] = g_m[n]
    MN = M * N
    X = np.fft.fft(x) / MN
    k = np.arange(-MN // 2, MN // 2)
    a = X[np.mod(k, MN)]
    t = 2 * np.pi * np.arange(L) / L
    textbook = np.real(np.exp(1j * np.outer(t, k)) @ a)
    assert rel(grid, textbook) < 1e-12


# ---------------------------------------------------------------- P10 -----------
def test_p10_2d_order_consistency_and_exactness():
    """Separable 2D: rows-first == columns-first, coarse-site
    consistency, and exact reconstruction of a 2D band-limited image."""
    Nn, scale = 8, 4
    bank = BANKS["f_df"]
    Lout = Nn * scale
    px = oracle.OraclePlan(2, Nn, Lout, bank)
    py = oracle.OraclePlan(2, Nn, Lout, bank)
    g = np.random.default_rng(10).standard_normal((2, 2, Nn, Nn))
    a = oracle.eval_2d(g, px, py, "rows_first")
    b = oracle.eval_2d(g, px, py, "cols_first")
    assert rel(a, b) < 1e-13
    assert np.max(np.abs(a[::scale, ::scale] - g[0, 0])) < 1e-12 * 10
    cols = oracle.eval_2d_columns(g, px, py, [0, 3, 31])
    assert rel(cols, a[:, [0, 3, 31]]) < 1e-13
    # band-limited real image with per-axis band -7..7 on a 32 x 32 grid
    rng = np.random.default_rng(12)
    C = rng.standard_normal((15, 15)) + 1j * rng.standard_normal((15, 15))
    C = C + np.conj(C[::-1, ::-1])                        # Hermitian => real image
    kk = np.arange(-7, 8)
    t = 2 * np.pi * np.arange(Lout) / Lout
    E = np.exp(1j * np.outer(t, kk))
    img = np.real(E @ C @ E.T)
    ch = synth.image_channels(img, Nn, bank)
    out = oracle.eval_2d(ch, px, py)
    assert rel(out, img) < 1e-12


# ---------------------------------------------------------------- misc ----------
def test_singular_bin_and_null_bin():
    """Example 3 / Remark 1: M = 1 Hilbert channel is
    singular at n = 0; declaring 0 a null bin zero-fills q(0)."""
    with pytest.raises(oracle.SingularBin) as e:
        oracle.OraclePlan(1, 8, 32, [("hilbert",)])
    assert e.value.n == 0
    P = oracle.OraclePlan(1, 8, 32, [("hilbert",)], null_bins=[0])
    assert np.all(P.Q[4] == 0)                           # n = 0 is index 0 - K1 = 4
    assert abs(P.Q[5][0, 0] - 1j) < 1e-15                # q = 1/(-i sgn 1) = i


def test_cfg1_exact_fp64():
    """Config 1 (BASELINE.json configs[0]): exact versus the closed form."""
    c = synth.CONFIGS[1]
    d = synth.cfg1()
    P = oracle.OraclePlan(c["M"], c["N"], c["L"], c["bank"])
    assert rel(P.eval(d["g"])[0], d["truth"][0]) < 1e-12


# ---------------------------------------------------------------- P11: SISR pipeline (NEXT-2)
def test_p11_sisr_consistency_constant_and_smooth():
    """oracle.sisr: (a) the identity channel is reproduced at the
    sample sites of both passes, so HR[3i][3j] = LR[i][j] exactly (Theorem consistency,
    PAPER.md:546-585); (b) a constant image stays constant; (c) for a smooth separable
    trig polynomial the centred differences are O(d^2)-accurate derivatives, so the
    output matches the true fine-grid image to that order (a wrong 2 pi / N derivative
    scaling, a sign or a swapped channel fails by O(1))."""
    rng = np.random.default_rng(11)
    H, W, s = 14, 18, 3
    lr = rng.standard_normal((H, W))
    hr = oracle.sisr(lr, s)
    assert hr.shape == (s * H, s * W)
    assert np.max(np.abs(hr[::s, ::s] - lr)) < 1e-10
    c = oracle.sisr(np.full((H, W), 2.5), s)
    assert np.max(np.abs(c - 2.5)) < 1e-10
    H, W = 40, 36
    x = np.arange(W) * 2 * np.pi / W
    y = np.arange(H) * 2 * np.pi / H
    f = lambda yy, xx: np.cos(yy[:, None] * 2 + 0.3) * np.sin(xx[None, :] + 0.1)
    out = oracle.sisr(f(y, x), s)
    xf = np.arange(s * W) * 2 * np.pi / (s * W)
    yf = np.arange(s * H) * 2 * np.pi / (s * H)
    truth = f(yf, xf)
    err = np.linalg.norm(out - truth) / np.linalg.norm(truth)
    assert err < 5e-3, err


# ---------------------------------------------------------------- P12: complex output, general band
@pytest.mark.parametrize("bank,K1", [
    ([("identity",), ("hilbert",)], -11),                  # Example 5's band -N..N+1 (N = 11)
    ([("identity",), ("derivative", 1)], -3),              # shifted band
    ([("delay", 0.0), ("delay", 0.4), ("delay", 1.1)], -20),
])
def test_p12_complex_exact_reconstruction(bank, K1):
    """Theorem 1 for complex f: any complex trig polynomial on the
    band [K1, K1 + MN) is reproduced exactly from its channel samples by eval_complex."""
    M = len(bank)
    N = 12
    L = 2 * M * N
    P = oracle.OraclePlan(M, N, L, bank, K1=K1)
    rng = np.random.default_rng(abs(K1) + M)
    k = np.arange(K1, K1 + M * N)
    a = rng.standard_normal(len(k)) + 1j * rng.standard_normal(len(k))
    tn = 2 * np.pi * np.arange(N) / N
    g = np.stack([(a * np.array([P.multiplier(m, kk) for kk in k])) @ np.exp(1j * np.outer(k, tn))
                  for m in range(M)])[None]
    tp = 2 * np.pi * np.arange(L) / L
    truth = a @ np.exp(1j * np.outer(k, tp))
    out = P.eval_complex(g)[0]
    assert np.linalg.norm(out - truth) / np.linalg.norm(truth) < 1e-11


def test_p12_example5_printed_kernel():
    """Example 5: M = 2, b = (1, -i sgn n), band -N..N+1, N + 1 samples;
    the paper prints y_1(t) = (cos((N+1)t) - cos(Nt) + cos t - 1) / (2 cos t - 2)."""
    Np = 9
    P = oracle.OraclePlan(2, Np + 1, 4 * (Np + 1), [("identity",), ("hilbert",)], K1=-Np)
    t = np.linspace(0.1, 6.0, 37)
    k = np.arange(-Np, Np + 2)
    y1 = (P.r[0] @ np.exp(1j * np.outer(k, t)))
    printed = (np.cos((Np + 1) * t) - np.cos(Np * t) + np.cos(t) - 1) / (2 * np.cos(t) - 2)
    assert np.max(np.abs(y1 - printed)) < 1e-12


# ---------------------------------------------------------------- P13: error analysis (NEXT-4)
def _shift_averaged_error(P, spec, k_lo):
    """(N/2 pi) int_0^{2 pi/N} ||f_tau - T_N f_tau||^2 dtau by brute force:
    for each tau, the channels of f_tau = f(. - tau) are sampled exactly, T_N f_tau's band
    coefficients come from oracle.band_spectrum, and Parseval gives the squared error.
    The integrand is a trig polynomial in tau with period 2 pi / N, so J > (support width)/N
    uniform points integrate it exactly."""
    n = np.arange(k_lo, k_lo + len(spec))
    J = len(spec) // P.N + 3
    tn = 2 * np.pi * np.arange(P.N) / P.N
    B = np.array([[P.multiplier(m, nn) for nn in n] for m in range(P.M)])
    acc = 0.0
    for j in range(J):
        tau = 2 * np.pi * j / (P.N * J)
        at = spec * np.exp(-1j * n * tau)                    # coefficients of f_tau
        g = (B * at) @ np.exp(1j * np.outer(n, tn))          # [M][N] channel samples
        k, ah = oracle.band_spectrum(P, g)
        full = dict(zip(n, at))
        err = sum(abs(full.get(kk, 0.0) - v) ** 2 for kk, v in zip(k, ah))
        err += sum(abs(v) ** 2 for nn, v in zip(n, at) if nn < P.K1 or nn >= P.K1 + P.MN)
        acc += err
    return np.sqrt(acc / J)


@pytest.mark.parametrize("bank", [[("identity",), ("derivative", 1)],
                                  [("identity",), ("derivative", 1), ("derivative", 2)],
                                  [("identity",), ("hilbert",)]])
def test_p13_averaged_error_matches_shift_average(bank):
    """Theorem error (Eq. averageerror) against the definition it comes
    from (shift-averaged L2 error), plus eps >= sqrt(oob), eps <= bound,
    and eps = 0 for band-limited f."""
    M, N = len(bank), 8
    P = oracle.OraclePlan(M, N, 4 * M * N, bank)
    rng = np.random.default_rng(M + 40)
    k_lo = P.K1 - 2 * N - 3
    spec = (rng.standard_normal(M * N + 5 * N) + 1j * rng.standard_normal(M * N + 5 * N)) / (
        1 + np.abs(np.arange(k_lo, k_lo + M * N + 5 * N)) / 4.0)
    eps, bound, oob = oracle.averaged_error(P, spec, k_lo)
    brute = _shift_averaged_error(P, spec, k_lo)
    assert abs(eps - brute) < 1e-9 * brute
    assert eps >= np.sqrt(oob) - 1e-12 and eps <= bound + 1e-9
    inband = spec.copy()
    n = np.arange(k_lo, k_lo + len(spec))
    inband[(n < P.K1) | (n >= P.K1 + P.MN)] = 0
    assert oracle.averaged_error(P, inband, k_lo)[0] == 0.0


def test_p13_consistency_residual():
    """Theorem consistency: residual ~0 for band-limited
    and for arbitrary data; a corrupted inverse entry is detected (> 1e-6)."""
    bank = [("identity",), ("derivative", 1), ("derivative", 2)]
    P = oracle.OraclePlan(3, 16, 96, bank)
    rng = np.random.default_rng(13)
    g = rng.standard_normal((3, 16)) * np.array([1.0, 4.0, 16.0])[:, None]
    assert oracle.consistency_residual(P, g) < 1e-10 * np.abs(g).max()
    P.r = P.r.copy()
    P.r[1, 5] += 1e-3
    assert oracle.consistency_residual(P, g) > 1e-6


def test_p13_bound_closed_forms():
    """Exact values of eps, bound and oob (Eq. averageerror / errorestimate, PAPER.md:722-747,
    DESIGN.md reading R12) worked by hand, so that a slip in the bound (Omega = sup|r| instead
    of sup|r|^2, a dropped factor M, sum_m Omega_m replaced by max) fails:
    (i) M = 1 identity channel: r = 1, Omega = 1, b = 1, so every out-of-band coefficient
        aliases onto one in-band bin with weight 1 + 1 and bound^2 = oob + 1 * 1 * oob:
        eps = bound = sqrt(2 oob).
    (ii) M = 2, (1, ik), N = 4, band -4..3, a(5) = 1 only.  H_j = [[1, ij], [1, i(j+N)]],
        det = iN, H_j^{-1} = (1/(iN)) [[i(j+N), -ij], [-1, 1]] (Eq. defH),
        so r_0(j) = (j+N)/N, r_0(j+N) = -j/N, r_1(j) = i/N, r_1(j+N) = -i/N.  n = 5 lies in
        block k = 3 of class j = -3: the weights are |r_0(-3) + 5i r_1(-3)|^2 = |1/4 - 5/4|^2 = 1
        and |r_0(1) + 5i r_1(1)|^2 = |3/4 + 5/4|^2 = 4 (reconstruction -e^{-3it} + 2e^{it}
        from the aliased samples e^{it_n}, 5i e^{it_n}), so eps^2 = 1 + 1 + 4 = 6.
        Omega_0 = sup|r_0|^2 = 1 (r_0(0) = 1), Omega_1 = 1/16, sum_m |b_m(5)|^2 = 1 + 25:
        bound^2 = 1 + 2 (1 + 1/16) 26 = 56.25, bound = 7.5."""
    P1 = oracle.OraclePlan(1, 8, 32, [("identity",)])
    rng = np.random.default_rng(131)
    k_lo = -20
    spec = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    eps, bound, oob = oracle.averaged_error(P1, spec, k_lo)
    n = np.arange(k_lo, k_lo + 40)
    oob_ref = np.sum(np.abs(spec[(n < -4) | (n >= 4)]) ** 2)
    assert abs(oob - oob_ref) < 1e-12 * oob_ref
    assert abs(eps - np.sqrt(2 * oob_ref)) < 1e-12 * eps
    assert abs(bound - np.sqrt(2 * oob_ref)) < 1e-12 * bound
    P2 = oracle.OraclePlan(2, 4, 16, [("identity",), ("derivative", 1)])
    eps, bound, oob = oracle.averaged_error(P2, np.array([1.0 + 0j]), 5)
    assert abs(oob - 1.0) < 1e-14
    assert abs(eps - np.sqrt(6.0)) < 1e-13
    assert abs(bound - 7.5) < 1e-13
