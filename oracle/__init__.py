"""fp64 CPU oracle for MCI (arXiv 1802.10291) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_1802_10291_b200) never imports it, and it never imports the product.

Thin ctypes wrapper around ``mci_oracle.c`` (plain C, fp64, OpenMP); every
formula lives in the C file with its PAPER.md citation.  The only arithmetic
here is the composition of two 1D passes for 2D (row pass then column pass,
Re after each pass: SURVEY.md §8(c) item 13), written as
plain loops over rows/columns calling the 1D oracle.

Parity pins for every function are in tests/test_oracle_pins.py; nothing here
is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mci_oracle.c")
_LIB = os.path.join(_HERE, "libmci_oracle.so")

KIND = {"identity": 0, "derivative": 1, "hilbert": 2, "delay": 3, "table": 4}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        vp = ctypes.c_void_p
        L.ora_inverse.argtypes = [i32, i64, i64, vp, vp, vp, vp, vp, i32, vp, P(d)]
        L.ora_inverse.restype = i32
        L.ora_r_from_q.argtypes = [i32, i64, i64, vp, vp]
        L.ora_r_from_q.restype = None
        L.ora_kernel_table.argtypes = [i32, i64, i64, i64, vp, i32, vp, i32]
        L.ora_kernel_table.restype = i32
        L.ora_eval_grid.argtypes = [i32, i64, i64, vp, i64, vp, vp, i32]
        L.ora_eval_grid.restype = i32
        L.ora_eval_grid_points.argtypes = [i32, i64, i64, vp, vp, i64, vp, vp, i32]
        L.ora_eval_grid_points.restype = i32
        L.ora_eval_offgrid.argtypes = [i32, i64, i64, vp, i32, vp, i64, vp, vp, i32]
        L.ora_eval_offgrid.restype = i32
        L.ora_delay_kernel_table.argtypes = [i32, i64, i64, vp]
        L.ora_delay_kernel_table.restype = i32
        L.ora_eval_delay_points.argtypes = [i32, i64, i64, vp, i64, vp, vp, i32]
        L.ora_eval_delay_points.restype = i32
        L.ora_multiplier.argtypes = [i32, i32, d, vp, i64, i64, P(d), P(d)]
        L.ora_multiplier.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _threads(threads):
    return int(threads if threads else (os.cpu_count() or 1))


class SingularBin(Exception):
    def __init__(self, n):
        super().__init__(f"H_n singular at n={n}")
        self.n = n


class OraclePlan:
    """Oracle for one band/bank: inverse tables, kernel tables, evaluation.

    M channels, N samples per channel at t_n = 2 pi n/N, band {K1..K1+MN-1}
    (default K1 = -MN/2), L output points at t_p = 2 pi p/L."""

    def __init__(self, M, N, L, bank, K1=None, null_bins=(), threads=None):
        self.M, self.N, self.L = int(M), int(N), int(L)
        self.MN = self.M * self.N
        self.K1 = -(self.MN // 2) if K1 is None else int(K1)
        self.bank = list(bank)
        self.threads = _threads(threads)
        assert len(self.bank) == self.M
        kinds = np.array([KIND[b[0]] for b in self.bank], dtype=np.int32)
        orders = np.array([int(b[1]) if b[0] == "derivative" else 0 for b in self.bank], dtype=np.int32)
        taus = np.array([float(b[1]) if b[0] == "delay" else 0.0 for b in self.bank], dtype=np.float64)
        self._tables = [np.ascontiguousarray(np.asarray(b[1], dtype=np.complex128).view(np.float64))
                        if b[0] == "table" else None for b in self.bank]
        tabptrs = (ctypes.c_void_p * self.M)(*[(_ptr(t).value if t is not None else None)
                                               for t in self._tables])
        nb = np.asarray(list(null_bins), dtype=np.int64)
        Q = np.zeros((self.N, self.M, self.M, 2), dtype=np.float64)
        cond = ctypes.c_double(0.0)
        rc = lib().ora_inverse(self.M, self.N, self.K1, _ptr(kinds), _ptr(orders), _ptr(taus),
                               ctypes.cast(tabptrs, ctypes.c_void_p), _ptr(nb) if len(nb) else None,
                               len(nb), _ptr(Q), ctypes.byref(cond))
        if rc < 0:
            raise ValueError("bad arguments")
        if rc > 0:
            raise SingularBin(self.K1 + rc - 1)
        self.cond_max = cond.value
        self.Q = Q[..., 0] + 1j * Q[..., 1]          # Q[n-K1][m][l] = q_{m,l}(n)
        r = np.zeros((self.M, self.MN, 2), dtype=np.float64)
        lib().ora_r_from_q(self.M, self.N, self.K1, _ptr(Q), _ptr(r))
        self._r = r
        self.r = r[..., 0] + 1j * r[..., 1]          # r[m][k-K1] = r_m(k)
        self._Y = {}

    # -- multipliers / kernel tables ------------------------------------------------
    def multiplier(self, m, k):
        re, im = ctypes.c_double(), ctypes.c_double()
        b = self.bank[m]
        t = self._tables[m]
        lib().ora_multiplier(KIND[b[0]], int(b[1]) if b[0] == "derivative" else 0,
                             float(b[1]) if b[0] == "delay" else 0.0,
                             _ptr(t) if t is not None else None, self.K1, int(k),
                             ctypes.byref(re), ctypes.byref(im))
        return complex(re.value, im.value)

    def kernel_table(self, hilbert=False):
        """Y[m][s] = Re (H^h y_m)(2 pi s/L)."""
        key = bool(hilbert)
        if key not in self._Y:
            Y = np.zeros((self.M, self.L), dtype=np.float64)
            rc = lib().ora_kernel_table(self.M, self.MN, self.K1, self.L, _ptr(self._r), int(key),
                                        _ptr(Y), self.threads)
            assert rc == 0
            self._Y[key] = Y
        return self._Y[key]

    # -- evaluation -------------------------------------------------------------------
    def eval(self, g, hilbert=False):
        """Re T_N f (or Re H T_N f) on all L points for rows g[R][M][N] (any float dtype)."""
        g = np.ascontiguousarray(np.asarray(g, dtype=np.float64).reshape(-1, self.M, self.N))
        Y = self.kernel_table(hilbert)
        out = np.zeros((g.shape[0], self.L), dtype=np.float64)
        rc = lib().ora_eval_grid(self.M, self.N, self.L, _ptr(Y), g.shape[0], _ptr(g), _ptr(out),
                                 self.threads)
        if rc != 0:
            raise ValueError("L must be a multiple of N for grid evaluation")
        return out

    def eval_points(self, g_row, p, hilbert=False):
        g = np.ascontiguousarray(np.asarray(g_row, dtype=np.float64).reshape(self.M, self.N))
        p = np.ascontiguousarray(np.asarray(p, dtype=np.int64))
        Y = self.kernel_table(hilbert)
        out = np.zeros(len(p), dtype=np.float64)
        rc = lib().ora_eval_grid_points(self.M, self.N, self.L, _ptr(Y), _ptr(g), len(p), _ptr(p),
                                        _ptr(out), self.threads)
        assert rc == 0
        return out

    def eval_complex(self, g):
        """T_N f on the L points, complex (no real part), for complex rows g[R][M][N]
        (SURVEY.md §8(f) NEXT-3, C2C): f(t_p) = (1/N) sum_m sum_n g_m[n] y_m(t_p - t_n) with
        the complex kernels y_m(t) = sum_k r_m(k) e^{ikt} (Eq. appxi operator PAPER.md:311,
        544; Theorem 1).  Direct sums (small sizes)."""
        g = np.asarray(g, dtype=np.complex128).reshape(-1, self.M, self.N)
        L, N = self.L, self.N
        assert L % N == 0
        s = np.arange(L)
        k = np.arange(self.K1, self.K1 + self.MN)
        Yc = self.r @ np.exp(2j * np.pi * np.mod(np.outer(k, s), L) / L)   # [M][L], y_m(2 pi s / L)
        out = np.zeros((g.shape[0], L), dtype=np.complex128)
        step = L // N
        for n in range(N):
            idx = (s - n * step) % L
            for m in range(self.M):
                out += g[:, m, n, None] * Yc[m, idx][None, :]
        return out / N

    def eval_offgrid(self, g_row, t, hilbert=False):
        g = np.ascontiguousarray(np.asarray(g_row, dtype=np.float64).reshape(self.M, self.N))
        t = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
        out = np.zeros(len(t), dtype=np.float64)
        lib().ora_eval_offgrid(self.M, self.N, self.K1, _ptr(self._r), int(bool(hilbert)), _ptr(g),
                               len(t), _ptr(t), _ptr(out), self.threads)
        return out


def delay_kernel_table(M, N, L):
    """Closed-form Re y_m on the L grid for the delay bank tau_m = 2 pi m/(MN)."""
    Y = np.zeros((M, L), dtype=np.float64)
    rc = lib().ora_delay_kernel_table(M, N, L, _ptr(Y))
    assert rc == 0
    return Y


def delay_eval_points(M, N, L, g_row, p, threads=None):
    """Re T_N f at output indices p for the delay bank (closed-form kernel)."""
    g = np.ascontiguousarray(np.asarray(g_row, dtype=np.float64).reshape(M, N))
    p = np.ascontiguousarray(np.asarray(p, dtype=np.int64))
    out = np.zeros(len(p), dtype=np.float64)
    rc = lib().ora_eval_delay_points(M, N, L, _ptr(g), len(p), _ptr(p), _ptr(out), _threads(threads))
    assert rc == 0
    return out


def eval_2d(g, plan_x: OraclePlan, plan_y: OraclePlan, order="rows_first"):
    """Separable MCI of one image, PAPER.md:869 ("each row ... then each column").

    g[My][Mx][Ny][Nx] are the tensor-bank channel images.
    Row pass: for each (my, ny) apply the 1D oracle along x over channels mx
    -> I[my][ny][Lx] (real part).  Column pass: for each px apply the 1D oracle
    along y over channels my -> out[Ly][Lx].  order="cols_first" does the two
    passes the other way round (pin P10)."""
    g = np.asarray(g, dtype=np.float64)
    My, Mx, Ny, Nx = g.shape
    assert (My, Ny) == (plan_y.M, plan_y.N) and (Mx, Nx) == (plan_x.M, plan_x.N)
    if order == "rows_first":
        inter = np.empty((My, Ny, plan_x.L))
        for my in range(My):
            rows = np.transpose(g[my], (1, 0, 2))            # [ny][mx][nx]
            inter[my] = plan_x.eval(rows)
        cols = np.transpose(inter, (2, 0, 1))                # [px][my][ny]
        out = plan_y.eval(cols)                              # [px][py]
        return out.T.copy()
    inter = np.empty((Mx, Nx, plan_y.L))
    for mx in range(Mx):
        cols = np.transpose(g[:, mx], (2, 0, 1))             # [nx][my][ny]
        inter[mx] = plan_y.eval(cols)                        # [nx][py]
    rows = np.transpose(inter, (2, 0, 1))                    # [py][mx][nx]
    return plan_x.eval(rows)                                 # [py][px]


def eval_2d_columns(g, plan_x: OraclePlan, plan_y: OraclePlan, px_list):
    """Output columns out[:, px] for the listed px only (sampled 2D parity)."""
    g = np.asarray(g, dtype=np.float64)
    My, Mx, Ny, Nx = g.shape
    px_list = np.asarray(px_list, dtype=np.int64)
    out = np.empty((plan_y.L, len(px_list)))
    inter = np.empty((len(px_list), My, Ny))
    for my in range(My):
        for ny in range(Ny):
            inter[:, my, ny] = plan_x.eval_points(g[my, :, ny, :], px_list)
    out[:] = plan_y.eval(inter).T
    return out


def sisr(lr, scale=3, threads=None):
    """Single-image super-resolution by MCI as the paper describes it (
    SURVEY.md §8(f) NEXT-2), fp64, periodic image model.

    "We first compute interpolation result for each row of image, and then apply
    interpolation for each column by using the same operations.  The derivatives of
    image are computed by three-point centered-difference formula" with the Example-2
    bank (f, f', f'').  On the grid t = 2 pi x / W, d = 2 pi / W:
    f' = (f[x+1] - f[x-1]) / (2 d), f'' = (f[x+1] - 2 f[x] + f[x-1]) / d^2 (periodic).
    Returns the [scale H][scale W] image (real part after each pass)."""
    lr = np.asarray(lr, dtype=np.float64)
    H, W = lr.shape
    bank = [("identity",), ("derivative", 1), ("derivative", 2)]
    px = OraclePlan(3, W, scale * W, bank, threads=threads)
    py = OraclePlan(3, H, scale * H, bank, threads=threads)

    def fd(a, axis, n):
        d = 2 * np.pi / n
        fp, fm = np.roll(a, -1, axis), np.roll(a, 1, axis)
        return np.stack([a, (fp - fm) / (2 * d), (fp - 2 * a + fm) / (d * d)])

    rows = np.transpose(fd(lr, 1, W), (1, 0, 2))          # [H][3][W]
    inter = px.eval(rows)                                  # [H][sW]
    cols = np.transpose(fd(inter, 0, H), (2, 0, 1))        # [sW][3][H]
    return px_py_out_t(py.eval(cols))                      # [sH][sW]


def px_py_out_t(out_cols):
    """Column-pass output [sW][sH] -> image [sH][sW]."""
    return np.ascontiguousarray(np.asarray(out_cols).T)


# ---------------------------------------------------------------- error analysis (NEXT-4)
def band_spectrum(P: OraclePlan, g):
    """Fourier coefficients of T_N f on the band from channel samples g[M][N] (real or complex):
    a^(k) = (1/N) sum_m r_m(k) sum_p g_m(t_p) e^{-ik t_p}  (Eq. DFTexpression).
    Returns (k, a^(k)) for k = K1 .. K1 + MN - 1."""
    g = np.asarray(g, dtype=np.complex128).reshape(P.M, P.N)
    k = np.arange(P.K1, P.K1 + P.MN)
    tp = 2 * np.pi * np.arange(P.N) / P.N
    E = np.exp(-1j * np.outer(k, tp))                       # [MN][N]
    return k, np.einsum("mk,mk->k", P.r, (g @ E.T)) / P.N  # sum_m r_m(k) G_m(k) / N


def consistency_residual(P: OraclePlan, g):
    """max_{m,n} |(T_N f * h_m)(t_n) - g_m(t_n)| (Theorem consistency, PAPER.md:546-585;
    SPEC.md:327-335): reconstruct a^, apply each multiplier b_m on the band, resample."""
    g = np.asarray(g, dtype=np.complex128).reshape(P.M, P.N)
    k, a = band_spectrum(P, g)
    tn = 2 * np.pi * np.arange(P.N) / P.N
    E = np.exp(1j * np.outer(k, tn))
    res = 0.0
    for m in range(P.M):
        b = np.array([P.multiplier(m, kk) for kk in k])
        res = max(res, float(np.max(np.abs((a * b) @ E - g[m]))))
    return res


def averaged_error(P: OraclePlan, spec, k_lo):
    """eps(f, N) of Theorem error (Eq. averageerror) for the true spectrum
    a(n), n = k_lo .. k_lo + len(spec) - 1 (zero elsewhere); I_k = {K1 + (k-1)N .. K1 + kN - 1}:
      eps^2 = sum_{n not in I^N} |a(n)|^2
            + sum_{k not in 1..M} sum_{n in I_k} |a(n)|^2 sum_{l=1}^M |sum_m r_m(n + (l-k)N) b_m(n)|^2.
    bound (Eq. errorestimate; DESIGN.md reading: Cauchy-Schwarz with Omega_m = sup_band |r_m|^2):
      bound^2 = sum_{n not in I^N} |a(n)|^2 + M (sum_m Omega_m) sum_{n not in I^N} sum_m |a(n) b_m(n)|^2.
    Returns (eps, bound, out_of_band_energy).  Direct loops (test infrastructure)."""
    spec = np.asarray(spec, dtype=np.complex128)
    M, N, K1 = P.M, P.N, P.K1
    omega = np.max(np.abs(P.r) ** 2, axis=1)
    e2 = oob = cs = 0.0
    for i, an in enumerate(spec):
        n = k_lo + i
        kb = (n - K1) // N + 1                               # block index of n
        if 1 <= kb <= M:
            continue
        a2 = abs(an) ** 2
        oob += a2
        b = np.array([P.multiplier(m, n) for m in range(M)])
        w = 0.0
        for l in range(1, M + 1):
            e = n + (l - kb) * N                             # the class's element in block l
            w += abs(np.sum(P.r[:, e - K1] * b)) ** 2
        e2 += a2 * (1.0 + w)
        cs += a2 * np.sum(np.abs(b) ** 2)
    return np.sqrt(e2), np.sqrt(oob + M * omega.sum() * cs), oob
