"""B200-native fast multichannel interpolation (MCI, arXiv 1802.10291).

Thin Python binding over the C ABI in ``include/mci.h`` (``libmci.so``, built
in-tree for sm_100a by ``_build.py``).  This module only marshals arguments:
every step of the hot path runs in the CUDA kernels behind the ABI.  There is
no CPU fallback -- if the library cannot be loaded, importing or calling
raises.  PyTorch is used only to hand device buffers and streams over.

Bank description: one tuple per channel,
    ("identity",) | ("derivative", order) | ("hilbert",) | ("delay", tau) | ("table", b[k-K1] complex array)
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# MCI_LIB: an experimental build of the same library (tools/build_variant.sh), A/B timing only
LIB_PATH = os.environ.get("MCI_LIB") or os.path.join(_PKG, "libmci.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "mci.h")

MCI_OK, MCI_E_ARG, MCI_E_BAND, MCI_E_ALIAS, MCI_E_SINGULAR, MCI_E_SIZE, MCI_E_CUDA, MCI_E_UNSUPPORTED = range(8)
MCI_F32, MCI_F64 = 0, 1
MCI_OUT_HILBERT = 1
MCI_OFFGRID = 2
MCI_COMPLEX = 4
MCI_ANALYSIS = 8
K1_DEFAULT = -(2 ** 63)
_KIND = {"identity": 0, "derivative": 1, "hilbert": 2, "delay": 3, "table": 4}
PATH_NAMES = {0: "fused", 1: "fourstep", 2: "2d", 3: "sisr"}


class MCIError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        msg = _lib_handle().mci_status_str(status).decode() if _lib is not None else str(status)
        super().__init__(f"{what}: {msg} (status {status})")


class _System(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("order", ctypes.c_int), ("tau", ctypes.c_double),
                ("table", ctypes.c_void_p)]


_lib = None


def _lib_handle():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint
        L.mci_plan_create.argtypes = [ctypes.POINTER(vp), i32, i64, i64, vp, vp, i32, i32, u32]
        L.mci_plan_create.restype = i32
        L.mci_plan_create_band.argtypes = [ctypes.POINTER(vp), i32, i64, i64, i64, vp, vp, i32, i32, u32]
        L.mci_plan_create_band.restype = i32
        L.mci_plan_create_2d.argtypes = [ctypes.POINTER(vp), i32, i64, vp, i32, i64, vp, i32, i32, u32]
        L.mci_plan_create_2d.restype = i32
        L.mci_plan_destroy.argtypes = [vp]
        L.mci_plan_destroy.restype = None
        L.mci_execute_1d.argtypes = [vp, i64, vp, vp, vp, vp]
        L.mci_execute_1d.restype = i32
        L.mci_execute_offgrid.argtypes = [vp, i64, vp, i64, vp, vp, vp, vp]
        L.mci_execute_offgrid.restype = i32
        L.mci_plan_create_sisr.argtypes = [ctypes.POINTER(vp), i64, i64, i32, i32]
        L.mci_plan_create_sisr.restype = i32
        L.mci_execute_sisr.argtypes = [vp, i64, vp, vp, vp]
        L.mci_execute_sisr.restype = i32
        L.mci_consistency_residual.argtypes = [vp, i64, vp, vp, vp]
        L.mci_consistency_residual.restype = i32
        L.mci_averaged_error.argtypes = [vp, i64, vp, i64, i64, vp, vp]
        L.mci_averaged_error.restype = i32
        L.mci_execute_2d.argtypes = [vp, i64, vp, vp, vp]
        L.mci_execute_2d.restype = i32
        L.mci_execute_1d_host.argtypes = [vp, i64, vp, vp, vp]
        L.mci_execute_1d_host.restype = i32
        L.mci_execute_2d_host.argtypes = [vp, i64, vp, vp]
        L.mci_execute_2d_host.restype = i32
        L.mci_plan_cond_max.argtypes = [vp]
        L.mci_plan_cond_max.restype = ctypes.c_double
        L.mci_last_singular_bin.argtypes = []
        L.mci_last_singular_bin.restype = i64
        L.mci_plan_workspace_bytes.argtypes = [vp]
        L.mci_plan_workspace_bytes.restype = ctypes.c_size_t
        L.mci_plan_path.argtypes = [vp]
        L.mci_plan_path.restype = i32
        L.mci_plan_launches.argtypes = [vp, i64]
        L.mci_plan_launches.restype = i64
        L.mci_status_str.argtypes = [i32]
        L.mci_status_str.restype = ctypes.c_char_p
        L.mci_version.argtypes = []
        L.mci_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def header_functions():
    """Function names declared in include/mci.h (for the ABI export test)."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mci_[a-z0-9_]+)\s*\(", txt)))


def _systems(bank):
    arr = (_System * len(bank))()
    keep = []
    for i, spec in enumerate(bank):
        kind = spec[0]
        arr[i].kind = _KIND[kind]
        arr[i].order = int(spec[1]) if kind == "derivative" else 0
        arr[i].tau = float(spec[1]) if kind == "delay" else 0.0
        if kind == "table":
            t = np.ascontiguousarray(np.asarray(spec[1], dtype=np.complex128).view(np.float64))
            keep.append(t)
            arr[i].table = t.ctypes.data
        else:
            arr[i].table = None
    return arr, keep


def _host_req(x, name, n_values, dtype, cplx=False):
    """Host buffers of the *_host entry points: C-contiguous, plan dtype, the expected size."""
    want = {("f32", False): "float32", ("f64", False): "float64",
            ("f32", True): "complex64", ("f64", True): "complex128"}[(dtype, bool(cplx))]
    if hasattr(x, "data_ptr"):  # CPU torch tensor
        if x.is_cuda or not x.is_contiguous() or str(x.dtype).split(".")[-1] != want or x.numel() != n_values:
            raise ValueError(f"{name}: contiguous CPU {want} tensor of {n_values} values required")
    else:
        if not (isinstance(x, np.ndarray) and x.flags.c_contiguous and x.dtype == np.dtype(want)
                and x.size == n_values):
            raise ValueError(f"{name}: C-contiguous {want} array of {n_values} values required")


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _req(t, name, dtype, shape=None, device=None):
    """Caller-supplied tensor checks (argument marshalling, not arithmetic): the C ABI takes raw
    pointers, so a wrong dtype, shape, device or a strided view would make the kernels read or
    write outside the buffer instead of failing."""
    if not t.is_cuda:
        raise ValueError(f"{name}: CUDA tensor required (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name}: contiguous tensor required")
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, plan needs {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")


def _check(status, what):
    if status != MCI_OK:
        if status == MCI_E_SINGULAR:
            raise MCIError(status, f"{what} (singular bin n={_lib_handle().mci_last_singular_bin()})")
        raise MCIError(status, what)


class Plan:
    """1D MCI plan: M channels x N samples -> L outputs (f, optionally Hf)."""

    def __init__(self, M, N, L, bank, null_bins=(), dtype="f32", hilbert=False, offgrid=False,
                 complex=False, K1=None, analysis=False):
        lib = _lib_handle()
        self.M, self.N, self.L = int(M), int(N), int(L)
        self.dtype = dtype
        self.hilbert = bool(hilbert)
        self.offgrid = bool(offgrid)
        self.complex = bool(complex)
        sys_arr, self._keep = _systems(bank)
        nb = np.ascontiguousarray(np.asarray(list(null_bins), dtype=np.int64))
        h = ctypes.c_void_p()
        flags = ((MCI_OUT_HILBERT if hilbert else 0) | (MCI_OFFGRID if offgrid else 0) |
                 (MCI_COMPLEX if complex else 0) | (MCI_ANALYSIS if analysis else 0))
        st = lib.mci_plan_create_band(ctypes.byref(h), self.M, self.N, self.L,
                                      K1_DEFAULT if K1 is None else int(K1), ctypes.addressof(sys_arr),
                                      nb.ctypes.data if len(nb) else None, len(nb),
                                      MCI_F64 if dtype == "f64" else MCI_F32, flags)
        _check(st, "mci_plan_create")
        self._h = h

    @property
    def path(self):
        return PATH_NAMES[_lib_handle().mci_plan_path(self._h)]

    @property
    def cond_max(self):
        return _lib_handle().mci_plan_cond_max(self._h)

    def launches(self, batch):
        return int(_lib_handle().mci_plan_launches(self._h, int(batch)))

    @property
    def workspace_bytes(self):
        return int(_lib_handle().mci_plan_workspace_bytes(self._h))

    def torch_dtype(self):
        import torch
        if self.complex:
            return torch.complex128 if self.dtype == "f64" else torch.complex64
        return torch.float64 if self.dtype == "f64" else torch.float32

    def execute(self, g, f=None, hf=None, stream=None):
        """g: CUDA tensor [batch][M][N] (contiguous, plan dtype).  Returns f (and hf)."""
        import torch
        _req(g, "g", self.torch_dtype())
        if g.dim() < 2 or tuple(g.shape[-2:]) != (self.M, self.N):
            raise ValueError(f"g: shape {tuple(g.shape)}, expected [batch][{self.M}][{self.N}]")
        batch = g.numel() // (self.M * self.N)
        if f is None:
            f = torch.empty((batch, self.L), dtype=g.dtype, device=g.device)
        _req(f, "f", g.dtype, (batch, self.L), g.device)
        if self.hilbert:
            if hf is None:
                hf = torch.empty((batch, self.L), dtype=g.dtype, device=g.device)
            _req(hf, "hf", g.dtype, (batch, self.L), g.device)
        st = _lib_handle().mci_execute_1d(self._h, batch, _dptr(g), _dptr(f), _dptr(hf) if self.hilbert else None,
                                          _stream(stream))
        _check(st, "mci_execute_1d")
        return (f, hf) if self.hilbert else f

    def execute_offgrid(self, g, t, f=None, hf=None, stream=None):
        """f(t_j) = Re T_N f(t_j) (and Hf) at arbitrary points t (CUDA tensor [n_pts], radians);
        plan created with offgrid=True.  Returns f [batch][n_pts] (and hf)."""
        import torch
        if not self.offgrid:
            raise ValueError("plan was not created with offgrid=True")
        _req(g, "g", self.torch_dtype())
        if g.dim() < 2 or tuple(g.shape[-2:]) != (self.M, self.N):
            raise ValueError(f"g: shape {tuple(g.shape)}, expected [batch][{self.M}][{self.N}]")
        if t.dim() != 1:
            raise ValueError("t: 1-D tensor of points required")
        _req(t, "t", g.dtype, device=g.device)
        batch = g.numel() // (self.M * self.N)
        npts = t.numel()
        if f is None:
            f = torch.empty((batch, npts), dtype=g.dtype, device=g.device)
        _req(f, "f", g.dtype, (batch, npts), g.device)
        if self.hilbert:
            if hf is None:
                hf = torch.empty((batch, npts), dtype=g.dtype, device=g.device)
            _req(hf, "hf", g.dtype, (batch, npts), g.device)
        st = _lib_handle().mci_execute_offgrid(self._h, batch, _dptr(g), npts, _dptr(t), _dptr(f),
                                               _dptr(hf) if self.hilbert else None, _stream(stream))
        _check(st, "mci_execute_offgrid")
        return (f, hf) if self.hilbert else f

    def consistency_residual(self, g, out=None, stream=None):
        """max_{m,n} |(T_N f * h_m)(t_n) - g_m[n]| per row (plan created with analysis=True)."""
        import torch
        _req(g, "g", self.torch_dtype())
        if g.dim() < 2 or tuple(g.shape[-2:]) != (self.M, self.N):
            raise ValueError(f"g: shape {tuple(g.shape)}, expected [batch][{self.M}][{self.N}]")
        batch = g.numel() // (self.M * self.N)
        if out is None:
            out = torch.empty((batch,), dtype=g.dtype, device=g.device)
        _req(out, "out", g.dtype, (batch,), g.device)
        _check(_lib_handle().mci_consistency_residual(self._h, batch, _dptr(g), _dptr(out), _stream(stream)),
               "mci_consistency_residual")
        return out

    def averaged_error(self, spec, k_lo, out=None, stream=None):
        """eps(f, N), its bound and the out-of-band energy per spectrum: spec complex CUDA tensor
        [batch][n_freq] holding a(k_lo .. k_lo + n_freq - 1).  Returns [batch][3]."""
        import torch
        cdt = torch.complex128 if self.dtype == "f64" else torch.complex64
        rdt = torch.float64 if self.dtype == "f64" else torch.float32
        _req(spec, "spec", cdt)
        if spec.dim() != 2:
            raise ValueError("spec: [batch][n_freq] required")
        batch, nf = spec.shape
        if out is None:
            out = torch.empty((batch, 3), dtype=rdt, device=spec.device)
        _req(out, "out", rdt, (batch, 3), spec.device)
        _check(_lib_handle().mci_averaged_error(self._h, batch, _dptr(spec), int(k_lo), nf, _dptr(out),
                                                _stream(stream)), "mci_averaged_error")
        return out

    def execute_host(self, g, f, hf=None):
        """Host buffers (numpy arrays or CPU tensors, ideally pinned): H2D, compute, D2H inside."""
        def p(x):
            return ctypes.c_void_p(x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data)
        batch = int(np.prod(g.shape)) // (self.M * self.N)
        _host_req(g, "g", batch * self.M * self.N, self.dtype, self.complex)
        _host_req(f, "f", batch * self.L, self.dtype, self.complex)
        if self.hilbert:
            _host_req(hf, "hf", batch * self.L, self.dtype, self.complex)
        st = _lib_handle().mci_execute_1d_host(self._h, batch, p(g), p(f), p(hf) if self.hilbert else None)
        _check(st, "mci_execute_1d_host")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mci_plan_destroy(h)
            self._h = None


class Plan2D:
    """Separable 2D MCI: channel images [n][My][Mx][Ny][Nx] -> [n][scale*Ny][scale*Nx]."""

    def __init__(self, Mx, Nx, bank_x, My, Ny, bank_y, scale, dtype="f32"):
        lib = _lib_handle()
        self.Mx, self.Nx, self.My, self.Ny, self.scale = int(Mx), int(Nx), int(My), int(Ny), int(scale)
        self.dtype = dtype
        sx, self._kx = _systems(bank_x)
        sy, self._ky = _systems(bank_y)
        h = ctypes.c_void_p()
        st = lib.mci_plan_create_2d(ctypes.byref(h), self.Mx, self.Nx, ctypes.addressof(sx), self.My, self.Ny,
                                    ctypes.addressof(sy), self.scale, MCI_F64 if dtype == "f64" else MCI_F32, 0)
        _check(st, "mci_plan_create_2d")
        self._h = h

    def launches(self, n):
        return int(_lib_handle().mci_plan_launches(self._h, int(n)))

    @property
    def workspace_bytes(self):
        return int(_lib_handle().mci_plan_workspace_bytes(self._h))

    def execute(self, g, out=None, stream=None):
        import torch
        dt = torch.float64 if self.dtype == "f64" else torch.float32
        _req(g, "g", dt)
        if g.numel() % (self.My * self.Mx * self.Ny * self.Nx):
            raise ValueError(f"g: {g.numel()} elements is not a whole number of [{self.My}][{self.Mx}][{self.Ny}][{self.Nx}] images")
        n = g.numel() // (self.My * self.Mx * self.Ny * self.Nx)
        if out is None:
            out = torch.empty((n, self.scale * self.Ny, self.scale * self.Nx), dtype=dt, device=g.device)
        _req(out, "out", dt, (n, self.scale * self.Ny, self.scale * self.Nx), g.device)
        st = _lib_handle().mci_execute_2d(self._h, n, _dptr(g), _dptr(out), _stream(stream))
        _check(st, "mci_execute_2d")
        return out

    def execute_host(self, g, out):
        def p(x):
            return ctypes.c_void_p(x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data)
        n = int(np.prod(g.shape)) // (self.My * self.Mx * self.Ny * self.Nx)
        _host_req(g, "g", n * self.My * self.Mx * self.Ny * self.Nx, self.dtype)
        _host_req(out, "out", n * self.scale * self.Ny * self.scale * self.Nx, self.dtype)
        st = _lib_handle().mci_execute_2d_host(self._h, n, p(g), p(out))
        _check(st, "mci_execute_2d_host")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mci_plan_destroy(h)
            self._h = None


def version():
    return _lib_handle().mci_version().decode()


class SisrPlan:
    """Single-image super-resolution by MCI: periodic H x W images ->
    scale*H x scale*W, rows then columns, channels f, f', f'' by three-point centred
    differences, Example-2 bank."""

    def __init__(self, H, W, scale=3, dtype="f32"):
        lib = _lib_handle()
        self.H, self.W, self.scale, self.dtype = int(H), int(W), int(scale), dtype
        h = ctypes.c_void_p()
        st = lib.mci_plan_create_sisr(ctypes.byref(h), self.H, self.W, self.scale,
                                      MCI_F64 if dtype == "f64" else MCI_F32)
        _check(st, "mci_plan_create_sisr")
        self._h = h

    def launches(self, n_images):
        return int(_lib_handle().mci_plan_launches(self._h, int(n_images)))

    def execute(self, lr, hr=None, stream=None):
        """lr: CUDA tensor [n][H][W] (plan dtype).  Returns hr [n][scale H][scale W]."""
        import torch
        dt = torch.float64 if self.dtype == "f64" else torch.float32
        _req(lr, "lr", dt)
        if lr.dim() < 2 or tuple(lr.shape[-2:]) != (self.H, self.W):
            raise ValueError(f"lr: shape {tuple(lr.shape)}, expected [n][{self.H}][{self.W}]")
        n = lr.numel() // (self.H * self.W)
        if hr is None:
            hr = torch.empty((n, self.scale * self.H, self.scale * self.W), dtype=dt, device=lr.device)
        _req(hr, "hr", dt, (n, self.scale * self.H, self.scale * self.W), lr.device)
        st = _lib_handle().mci_execute_sisr(self._h, n, _dptr(lr), _dptr(hr), _stream(stream))
        _check(st, "mci_execute_sisr")
        return hr

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mci_plan_destroy(h)
            self._h = None

