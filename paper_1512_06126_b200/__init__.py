"""emie-b200: the CIE operator apply, Green's-tensor build and FGMRES of the
reference `emie` library (arXiv:1512.06126), rebuilt for B200 (sm_100a).

This Python package mirrors the reference's public C++ API
(/root/reference/proj/include/emie/*.hpp, namespace emie) over the C ABI in
include/emie_cu.h (libemie_cu.so, built in-tree by build.py). Names,
argument meaning and error behaviour follow the reference so that parity
tests read like its own tests:

    model = LayeredModel(tops=[0, 400], sigma=[0, 0.01, 0.1])
    grid = make_grid(model, breaks, nx, ny, hx, hy, x0, y0)
    sop = assemble_operator(grid, model, omega)      # device Green's build
    w = apply(sop, v)                                # toeplitz.hpp:43
    sys = build_system(grid, sop)                    # cie.hpp:36
    u, rep = solve_cie(grid, model, sop, rhs, SolverConfig(tol=1e-6))

Fields may be numpy arrays (host; copied in and out) or torch complex128
CUDA tensors (device-resident; no copies). There is no CPU fallback: every
compute call goes through libemie_cu.so and raises if it cannot be loaded.

Exceptions map the reference's: std::invalid_argument -> InvalidArgument
(ValueError), std::domain_error -> DomainError (ArithmeticError),
std::out_of_range -> OutOfRange (IndexError), std::runtime_error ->
EmieRuntimeError (RuntimeError).
"""
from __future__ import annotations

import bisect
import ctypes
import os as _os
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "LayeredModel", "AnomalyGrid", "make_grid", "fill_box", "smooth_embedding_size",
    "SpectralOperator", "SystemOperator", "transform_operator", "assemble_operator",
    "apply", "build_system", "SolverConfig", "SolveReport", "fgmres_system", "solve_cie",
    "contrast_coefficients", "FilterParams", "design_offset_filters",
    "InvalidArgument", "DomainError", "OutOfRange", "EmieRuntimeError", "CudaError", "lib",
]

_PKG = Path(__file__).resolve().parent
_LIB_PATH = _PKG / "libemie_cu.so"
if _os.environ.get("EMIE_CU_LIBRARY"):  # developer override (kernel experiments)
    _LIB_PATH = Path(_os.environ["EMIE_CU_LIBRARY"]).resolve()
SIGMA_FLOOR = 1e-9  # include/emie/layered.hpp:32
MU0 = 1.2566370614359172e-06


class InvalidArgument(ValueError):
    pass


class DomainError(ArithmeticError):
    pass


class OutOfRange(IndexError):
    pass


class EmieRuntimeError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_EXC = {1: InvalidArgument, 2: DomainError, 3: OutOfRange, 4: EmieRuntimeError, 5: CudaError}

_lib = None


class _Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("iterations", ctypes.c_int),
                ("residual", ctypes.c_double), ("history_len", ctypes.c_int)]


def lib():
    """Load libemie_cu.so (building it first if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        from . import build as _b
        _b.build()
    L = ctypes.CDLL(str(_LIB_PATH))
    vp, dp, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
    L.emie_cu_last_error.restype = ctypes.c_char_p
    L.emie_cu_version.restype = ctypes.c_char_p
    L.emie_cu_launch_count.restype = ctypes.c_longlong
    sig = {
        "emie_cu_smooth_embedding_size": [ctypes.c_int, ip],
        "emie_cu_operator_from_blocks": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         vp, ctypes.POINTER(vp), vp],
        "emie_cu_greens_build": [ctypes.c_int, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, ctypes.c_int,
                                 ctypes.POINTER(vp), vp],
        "emie_cu_operator_dims": [vp, ip, dp],
        "emie_cu_greens_offsets": [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ip, ctypes.c_int,
                                   ip],
        "emie_cu_greens_blocks": [ctypes.c_int, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, ctypes.c_int,
                                  ctypes.c_int, vp, vp],
        "emie_cu_operator_from_greens_blocks": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_double, vp, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(vp), vp],
        "emie_cu_vec_dots": [vp, ctypes.c_longlong, ctypes.c_int, vp, ctypes.c_longlong, ctypes.c_int, vp, vp],
        "emie_cu_vec_update": [vp, vp, ctypes.c_longlong, ctypes.c_int, vp, ctypes.c_longlong, vp, vp, vp],
        "emie_cu_vec_dcgs_dots": [vp, ctypes.c_longlong, ctypes.c_int, vp, ctypes.c_longlong, vp, vp],
        "emie_cu_vec_dcgs_update": [vp, vp, ctypes.c_longlong, ctypes.c_int, vp, ctypes.c_longlong, vp, vp],
        "emie_cu_vec_combine": [vp, vp, ctypes.c_longlong, ctypes.c_int, vp, ctypes.c_longlong, vp],
        "emie_cu_vec_scale": [vp, vp, ctypes.c_double, ctypes.c_longlong, vp],
        "emie_cu_vec_residual": [vp, vp, vp, ctypes.c_longlong, vp, vp],
        "emie_cu_operator_xy_symmetry": [vp, ctypes.c_int, ip],
        "emie_cu_operator_download_spectra": [vp, vp],
        "emie_cu_operator_download_blocks": [vp, vp],
        "emie_cu_design_offset_filters": [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          vp, vp, vp],
        "emie_cu_apply_spectral": [vp, vp, vp, ctypes.c_int, vp],
        "emie_cu_system_create": [vp, vp, vp, vp, ctypes.POINTER(vp)],
        "emie_cu_system_download": [vp, vp, vp, vp],
        "emie_cu_apply_system": [vp, vp, vp, ctypes.c_int, vp],
        "emie_cu_apply_system_host": [vp, vp, vp, ctypes.c_int, vp],
        "emie_cu_fgmres": [vp, vp, vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(_Report), vp, ctypes.c_int, vp],
        "emie_cu_device_count": [ip],
        "emie_cu_pool_reserve": [ctypes.c_ulonglong],
        "emie_cu_receiver_fields": [ctypes.c_int, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, vp, vp, ctypes.c_int, vp, ctypes.c_int, vp, vp],
        "emie_cu_receiver_tensors": [ctypes.c_int, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, vp, vp, ctypes.c_int, ctypes.c_int, vp],
        "emie_cu_fgmres_ex": [vp, vp, vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(_Report), vp, ctypes.c_int, vp, vp, vp],
        "emie_cu_fgmres_map": [ctypes.c_longlong, ctypes.c_int, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_double,
                               ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Report), vp, ctypes.c_int, vp],
        "emie_cu_dense_apply": [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp],
        "emie_cu_assemble_blocks": [ctypes.c_int, vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, ctypes.c_int, vp, vp, vp],
        "emie_cu_vfunctions": [ctypes.c_int, vp, vp, ctypes.c_int, vp, ctypes.c_double, ctypes.c_int, vp, vp],
        "emie_cu_kernel_output": [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, vp],
        # sharded apply (distributed.py)
        "emie_cu_geometry_create": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
        "emie_cu_operator_restrict_modes": [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
        "emie_cu_mode_list": [vp, ctypes.c_int, ctypes.c_int, ip, ctypes.c_int, ip],
        "emie_cu_operator_shard_octant": [vp, ctypes.c_int, ip],
        "emie_cu_lateral_forward": [vp, vp, vp, vp, ctypes.c_int, vp],
        "emie_cu_lateral_inverse": [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp],
        "emie_cu_contract_modes": [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp],
        "emie_cu_move_planes": [vp, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_longlong, ip, ip,
                                ctypes.c_int, vp],
        # peer-memory exchange (distributed.PeerExchange)
        "emie_cu_peer_alloc": [ctypes.c_size_t, ctypes.POINTER(vp)],
        "emie_cu_peer_free": [vp],
        "emie_cu_ipc_handle": [vp, vp],
        "emie_cu_ipc_open": [vp, ctypes.POINTER(vp)],
        "emie_cu_ipc_close": [vp],
        "emie_cu_peer_signal": [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.c_int, vp],
        "emie_cu_peer_wait": [vp, ctypes.c_int, ctypes.c_int, vp],
        "emie_cu_peer_status": [ip],
        "emie_cu_lateral_forward_peer": [vp, vp, vp, vp, ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, vp],
        "emie_cu_lateral_forward_peer_supported": [vp, ip],
        "emie_cu_lateral_forward_peer_split": [vp, vp, vp, ip, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_int, vp],
        "emie_cu_contract_modes_peer": [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp), ip,
                                        ctypes.c_int, vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.emie_cu_operator_destroy.argtypes = [vp]
    L.emie_cu_operator_destroy.restype = None
    L.emie_cu_system_destroy.argtypes = [vp]
    L.emie_cu_system_destroy.restype = None
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        msg = lib().emie_cu_last_error().decode(errors="replace")
        raise _EXC.get(rc, EmieRuntimeError)(msg)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _stream_of(t=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def smooth_embedding_size(n: int) -> int:
    """include/emie/toeplitz.hpp:13 (src/toeplitz.cpp:18-26)."""
    out = ctypes.c_int(0)
    _check(lib().emie_cu_smooth_embedding_size(int(n), ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------------ model ---
@dataclass
class LayeredModel:
    """include/emie/layered.hpp:15-33. Layer 0 is the upper halfspace (air)."""
    tops: Sequence[float]
    sigma: Sequence[complex]

    def layer_count(self) -> int:
        return len(self.sigma)

    def layer_of(self, z: float) -> int:  # layered.cpp:32-36
        return bisect.bisect_right(list(self.tops), z)

    def top_of(self, m: int) -> float:  # layered.cpp:38
        return self.tops[0] if m == 0 else self.tops[m - 1]

    def bottom_of(self, m: int) -> float:  # layered.cpp:40-43
        return self.tops[-1] if m == len(self.tops) else self.tops[m]

    def thickness(self, m: int) -> float:
        return self.bottom_of(m) - self.top_of(m)

    def sigma_floored(self, m: int) -> complex:  # layered.cpp:47-51
        s = complex(self.sigma[m])
        return complex(SIGMA_FLOOR, s.imag) if s.real < SIGMA_FLOOR else s

    def validate(self) -> None:  # layered.cpp:53-65
        if len(self.tops) == 0:
            raise InvalidArgument("layered model needs at least one interface")
        if len(self.sigma) != len(self.tops) + 1:
            raise InvalidArgument("layered model: sigma count must be tops count + 1")
        for a, b in zip(self.tops, self.tops[1:]):
            if not a < b:
                raise InvalidArgument("layered model: interface depths must increase")
        if not all(math.isfinite(d) for d in self.tops):
            raise InvalidArgument("layered model: non-finite depth")
        for s in self.sigma:
            s = complex(s)
            if not (math.isfinite(s.real) and math.isfinite(s.imag)):
                raise InvalidArgument("layered model: non-finite conductivity")


def _partition(model: LayeredModel, breaks):
    """VerticalPartition::create (src/layered.cpp:191-208)."""
    if len(breaks) < 2:
        raise InvalidArgument("vertical partition needs at least one interval")
    L = len(model.tops)
    layer = []
    for i in range(len(breaks) - 1):
        if not breaks[i] < breaks[i + 1]:
            raise InvalidArgument("vertical partition: breaks must increase")
        m = model.layer_of(breaks[i])
        slack = 1e-7 * (1.0 + abs(breaks[i + 1]))
        if m < L and breaks[i + 1] > model.bottom_of(m) + slack:
            raise InvalidArgument("vertical partition: interval straddles a layer interface")
        layer.append(m)
    return layer


@dataclass
class AnomalyGrid:
    """include/emie/greens.hpp:22-38."""
    nx: int
    ny: int
    hx: float
    hy: float
    x0: float
    y0: float
    breaks: list
    layer: list
    sigma_a: np.ndarray  # (nz, ny, nx) complex
    sigma_b: np.ndarray  # (nz,) complex

    @property
    def nz(self) -> int:
        return len(self.layer)

    def dz(self, iz: int) -> float:
        return self.breaks[iz + 1] - self.breaks[iz]

    def volume(self, iz: int) -> float:  # greens.hpp:35
        return self.hx * self.hy * self.dz(iz)

    def validate(self, model: LayeredModel) -> None:  # greens.cpp:18-35
        if self.nx <= 0 or self.ny <= 0 or self.nz <= 0:
            raise InvalidArgument("grid: empty dimensions")
        if not (self.hx > 0.0) or not (self.hy > 0.0):
            raise InvalidArgument("grid: cell sizes must be positive")
        if self.sigma_a.size != self.nx * self.ny * self.nz or self.sigma_b.size != self.nz:
            raise InvalidArgument("grid: conductivity array sizes")
        if np.any(~(self.sigma_a.real >= 0.0)):
            raise InvalidArgument("grid: cell conductivity with negative real part")
        for m in self.layer:
            if not complex(model.sigma[m]).real > 0.0:
                raise InvalidArgument("grid: interval in a non-conducting layer; the anomaly must be "
                                      "buried in the conductive section")


def make_grid(model: LayeredModel, breaks, nx, ny, hx, hy, x0=0.0, y0=0.0) -> AnomalyGrid:
    """include/emie/greens.hpp:43-45 (src/greens.cpp:37-57)."""
    breaks = [float(b) for b in breaks]
    layer = _partition(model, breaks)
    sb = np.array([model.sigma_floored(m) for m in layer], dtype=np.complex128)
    sa = np.broadcast_to(sb[:, None, None], (len(layer), max(ny, 0), max(nx, 0))).copy()
    g = AnomalyGrid(int(nx), int(ny), float(hx), float(hy), float(x0), float(y0), breaks, layer, sa, sb)
    g.validate(model)
    return g


def fill_box(grid: AnomalyGrid, ix0, ix1, iy0, iy1, iz0, iz1, sigma) -> None:
    """include/emie/greens.hpp:48-49 (src/greens.cpp:59-67); inclusive box."""
    if (ix0 < 0 or iy0 < 0 or iz0 < 0 or ix1 >= grid.nx or iy1 >= grid.ny or iz1 >= grid.nz
            or ix0 > ix1 or iy0 > iy1 or iz0 > iz1):
        raise InvalidArgument("fill_box: index box out of range")
    grid.sigma_a[iz0:iz1 + 1, iy0:iy1 + 1, ix0:ix1 + 1] = sigma


# -------------------------------------------------------------- operators ---
@dataclass
class FilterParams:
    """include/emie/hankel.hpp:20-26."""
    step: float = 0.2
    shift: float = 0.0964
    half: int = 512
    n1: int = -250
    n2: int = 200

    def as_array(self) -> np.ndarray:
        return np.array([self.step, self.shift, self.half, self.n1, self.n2], dtype=np.float64)


class SpectralOperator:
    """include/emie/toeplitz.hpp:21-35, device-resident (handle to the C ABI
    operator). `comp` downloads the six reference component arrays."""

    def __init__(self, handle):
        self._h = handle
        dims = (ctypes.c_int * 7)()
        om = ctypes.c_double(0.0)
        _check(lib().emie_cu_operator_dims(self._h, dims, ctypes.byref(om)))
        self.nx, self.ny, self.nz, self.ex, self.ey, self.qx, self.qy = list(dims)
        self.omega = om.value

    @property
    def handle(self):
        return self._h

    def mode_count(self) -> int:
        return self.qx * self.qy

    def stored_complex_count(self) -> int:  # toeplitz.cpp:86-90
        return self.mode_count() * 2 * self.nz * (2 * self.nz + 1)

    @property
    def comp(self):
        flat = np.empty(self.stored_complex_count(), np.complex128)
        _check(lib().emie_cu_operator_download_spectra(self._h, _ptr(flat)))
        ntri, nfull, nm = self.nz * (self.nz + 1) // 2, self.nz * self.nz, self.mode_count()
        out, o = [], 0
        for c in range(6):
            n = nm * (ntri if c < 4 else nfull)
            out.append(flat[o:o + n])
            o += n
        return out

    def blocks(self) -> np.ndarray:
        """compressed operator blocks (ny, nx, 2nz(2nz+1)) when kept."""
        b = np.empty((self.ny, self.nx, 2 * self.nz * (2 * self.nz + 1)), np.complex128)
        _check(lib().emie_cu_operator_download_blocks(self._h, _ptr(b)))
        return b

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.emie_cu_operator_destroy(h)
            self._h = None


def transform_operator(blocks, nx: int, ny: int, nz: int, omega: float = 0.0) -> SpectralOperator:
    """include/emie/toeplitz.hpp:37 from a compressed operator given as the
    offset-major block array (ny, nx, 2nz(2nz+1)) in GreensBlock order."""
    b = _c128(blocks)
    if b.size != nx * ny * 2 * nz * (2 * nz + 1):
        raise InvalidArgument("transform_operator: block array size")
    h = ctypes.c_void_p()
    _check(lib().emie_cu_operator_from_blocks(int(nx), int(ny), int(nz), float(omega), _ptr(b),
                                              ctypes.byref(h), None))
    return SpectralOperator(h)


def assemble_operator(grid: AnomalyGrid, model: LayeredModel, omega: float,
                      params: Optional[FilterParams] = None, keep_blocks: bool = False) -> SpectralOperator:
    """assemble_operator + transform_operator (greens.hpp:144-147,
    toeplitz.hpp:37) as one device-resident build."""
    model.validate()
    grid.validate(model)
    tops = np.ascontiguousarray(model.tops, dtype=np.float64)
    sig = _c128(model.sigma)
    br = np.ascontiguousarray(grid.breaks, dtype=np.float64)
    fp = (params or FilterParams()).as_array()
    h = ctypes.c_void_p()
    _check(lib().emie_cu_greens_build(len(tops), _ptr(tops), _ptr(sig), grid.nz, _ptr(br), grid.nx,
                                      grid.ny, grid.hx, grid.hy, float(omega), _ptr(fp),
                                      int(keep_blocks), ctypes.byref(h), None))
    return SpectralOperator(h)


def assemble_block(grid: AnomalyGrid, model: LayeredModel, omega: float, offset_i, offset_j,
                   params: Optional[FilterParams] = None) -> np.ndarray:
    """assemble_block (greens.hpp:129-135) at one or more signed offsets, on
    the device -> (n, 2nz(2nz+1)) blocks in GreensBlock order (xx yy zz xy
    triangles, xz yz full); OutOfRange outside the grid (greens.cpp:153-154)."""
    model.validate()
    grid.validate(model)
    oi = np.ascontiguousarray(np.atleast_1d(offset_i), dtype=np.int32)
    oj = np.ascontiguousarray(np.atleast_1d(offset_j), dtype=np.int32)
    if oi.shape != oj.shape:
        raise InvalidArgument("assemble_block: offset arrays differ in length")
    tops = np.ascontiguousarray(model.tops, dtype=np.float64)
    sig = _c128(model.sigma)
    br = np.ascontiguousarray(grid.breaks, dtype=np.float64)
    fp = (params or FilterParams()).as_array()
    nz = grid.nz
    out = np.zeros((oi.size, 2 * nz * (2 * nz + 1)), np.complex128)
    _check(lib().emie_cu_assemble_blocks(len(tops), _ptr(tops), _ptr(sig), nz, _ptr(br), grid.nx, grid.ny,
                                         grid.hx, grid.hy, float(omega), _ptr(fp), oi.size,
                                         oi.ctypes.data_as(ctypes.c_void_p), oj.ctypes.data_as(ctypes.c_void_p),
                                         _ptr(out)))
    return out


def greens_offsets(nx: int, ny: int, hx: float, hy: float) -> np.ndarray:
    """Offsets oi*nx + oj the Green's build computes (the rest are x <-> y
    mirrors on square grids with hx == hy); the sharded build splits these."""
    L = lib()
    n = ctypes.c_int()
    _check(L.emie_cu_greens_offsets(int(nx), int(ny), float(hx), float(hy), None, 0, ctypes.byref(n)))
    out = np.zeros(max(1, n.value), np.int32)
    _check(L.emie_cu_greens_offsets(int(nx), int(ny), float(hx), float(hy),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n.value, ctypes.byref(n)))
    return out[:n.value]


def greens_blocks(grid: AnomalyGrid, model: LayeredModel, omega: float, c0: int, c1: int, d_blocks,
                  params: Optional[FilterParams] = None) -> None:
    """Blocks of computed offsets [c0, c1) (greens_offsets order) into the
    complex128 CUDA tensor d_blocks (ny, nx, 2nz(2nz+1)); other offsets untouched."""
    model.validate()
    grid.validate(model)
    tops = np.ascontiguousarray(model.tops, dtype=np.float64)
    sig = _c128(model.sigma)
    br = np.ascontiguousarray(grid.breaks, dtype=np.float64)
    fp = (params or FilterParams()).as_array()
    _check(lib().emie_cu_greens_blocks(len(tops), _ptr(tops), _ptr(sig), grid.nz, _ptr(br), grid.nx, grid.ny,
                                       grid.hx, grid.hy, float(omega), _ptr(fp), int(c0), int(c1),
                                       ctypes.c_void_p(d_blocks.data_ptr()), _stream_of(d_blocks)))


def operator_from_greens_blocks(grid: AnomalyGrid, omega: float, d_blocks, q0: int = 0,
                                q1: int = -1) -> SpectralOperator:
    """Mirror + transform_operator of quadrant modes [q0, q1) from the summed
    computed blocks (d_blocks is completed in place)."""
    h = ctypes.c_void_p()
    _check(lib().emie_cu_operator_from_greens_blocks(grid.nx, grid.ny, grid.nz, float(omega), grid.hx, grid.hy,
                                                     ctypes.c_void_p(d_blocks.data_ptr()), int(q0), int(q1),
                                                     ctypes.byref(h), _stream_of(d_blocks)))
    return SpectralOperator(h)


def warmup(reserve_bytes: int = 0) -> None:
    """Library initialisation: one tiny Green's build (16 x 16 x 2) and system
    apply, so the device code of the build and the first allocations of the
    stream-ordered pool are in place before a timed build (CUDA loads kernels
    lazily, on first launch); reserve_bytes > 0 also grows the library's
    memory pool by that much (emie_cu_pool_reserve)."""
    if reserve_bytes > 0:
        _check(lib().emie_cu_pool_reserve(ctypes.c_ulonglong(int(reserve_bytes))))
    model = LayeredModel([0.0, 1000.0], [0.0, 0.01, 0.1])
    grid = make_grid(model, [1100.0, 1200.0, 1300.0], 16, 16, 100.0, 100.0)
    op = assemble_operator(grid, model, 2.0 * np.pi)
    apply(build_system(grid, op), np.ones(3 * 16 * 16 * 2, np.complex128))


def restrict_modes(op: SpectralOperator, q0: int, q1: int) -> SpectralOperator:
    """A device copy of op holding only quadrant modes [q0, q1) (the mode
    shard of a sharded apply, distributed.py)."""
    h = ctypes.c_void_p()
    _check(lib().emie_cu_operator_restrict_modes(op.handle, int(q0), int(q1), ctypes.byref(h)))
    return SpectralOperator(h)


def xy_symmetric(op: SpectralOperator, disable: bool = False) -> bool:
    """True when the contraction runs on the octant modes only (the operator's
    blocks are exactly x <-> y symmetric on a square grid). disable=True turns
    the octant contraction off for this operator."""
    out = ctypes.c_int()
    _check(lib().emie_cu_operator_xy_symmetry(op.handle, int(bool(disable)), ctypes.byref(out)))
    return bool(out.value)


def mode_list(op: SpectralOperator, q0: int, q1: int) -> np.ndarray:
    """Full modes (mx*ey + my) of quadrant modes [q0, q1) in contraction order."""
    L = lib()
    n = ctypes.c_int()
    _check(L.emie_cu_mode_list(op.handle, int(q0), int(q1), None, 0, ctypes.byref(n)))
    out = np.zeros(max(1, n.value), np.int32)
    _check(L.emie_cu_mode_list(op.handle, int(q0), int(q1),
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n.value, ctypes.byref(n)))
    return out[:n.value]


def design_offset_filters(oi: int, oj: int, hx: float, hy: float,
                          params: Optional[FilterParams] = None):
    """Six filter weight sets of one offset (greens.cpp:133-140) -> (w[6, n], lam[n])."""
    p = params or FilterParams()
    n = max(1, p.n2 - p.n1 + 1)
    w = np.empty((6, n), np.float64)
    lam = np.empty(n, np.float64)
    fp = p.as_array()
    _check(lib().emie_cu_design_offset_filters(int(oi), int(oj), float(hx), float(hy), _ptr(fp),
                                               _ptr(w), _ptr(lam)))
    return w, lam


def vfunctions(model: LayeredModel, breaks, omega: float, lam) -> np.ndarray:
    """V-functions of every interval pair at the given lambdas as the device
    build evaluates them (layered.cpp:397-408) -> (n, 4, nz, nz) complex:
    V1, V1 + V3, V2 + V5 (upper triangle), V4 (full)."""
    model.validate()
    tops = np.ascontiguousarray(model.tops, dtype=np.float64)
    sig = _c128(model.sigma)
    br = np.ascontiguousarray(breaks, dtype=np.float64)
    lam = np.ascontiguousarray(np.atleast_1d(lam), dtype=np.float64)
    nz = len(br) - 1
    out = np.zeros((lam.size, 4, nz, nz), np.complex128)
    _check(lib().emie_cu_vfunctions(len(tops), _ptr(tops), _ptr(sig), nz, _ptr(br), float(omega), lam.size,
                                    _ptr(lam), _ptr(out)))
    return out


def receiver_tensors(grid: AnomalyGrid, model: LayeredModel, omega: float, receiver, ix: int, iy: int,
                     params: Optional[FilterParams] = None) -> np.ndarray:
    """int_cell G^E(M, M0) dM0 and int_cell G^H(M, M0) dM0 (SPEC.md
    receiver_green_integrals; paper Appendix A Eq. geh / Ge2) for the receiver
    M = (x, y, z) and every cell of column (ix, iy), on the device ->
    (nz, 2, 3, 3) complex: [k, 0] = G^E, [k, 1] = G^H, row = field component."""
    model.validate()
    grid.validate(model)
    tops = np.ascontiguousarray(model.tops, dtype=np.float64)
    sig = _c128(model.sigma)
    br = np.ascontiguousarray(grid.breaks, dtype=np.float64)
    fp = (params or FilterParams()).as_array()
    rec = np.ascontiguousarray(receiver, dtype=np.float64).reshape(3)
    out = np.zeros((grid.nz, 2, 3, 3), np.complex128)
    _check(lib().emie_cu_receiver_tensors(len(tops), _ptr(tops), _ptr(sig), grid.nz, _ptr(br), grid.nx, grid.ny,
                                          grid.hx, grid.hy, grid.x0, grid.y0, float(omega), _ptr(fp), _ptr(rec),
                                          int(ix), int(iy), _ptr(out)))
    return out


def receiver_fields(grid: AnomalyGrid, model: LayeredModel, omega: float, U, receivers,
                    params: Optional[FilterParams] = None) -> np.ndarray:
    """Anomalous receiver fields of CIE solutions (SPEC.md reconstruct_fields,
    paper Eq. APR_lab): sum_n (sigma_a - sigma_b) E_n int_n G dOmega with E_n =
    U_n / a_n. U: (nrhs, 3N) solutions; receivers (nrec, 3) -> (nrec, nrhs, 2, 3)
    complex: [., ., 0] = E, [., ., 1] = H (add the normal field for totals)."""
    model.validate()
    grid.validate(model)
    tops = np.ascontiguousarray(model.tops, dtype=np.float64)
    sig = _c128(model.sigma)
    br = np.ascontiguousarray(grid.breaks, dtype=np.float64)
    fp = (params or FilterParams()).as_array()
    u = _c128(U)
    ncell = grid.nx * grid.ny * grid.nz
    if u.size % (3 * ncell) != 0 or u.size == 0:
        raise InvalidArgument("receiver_fields: field shape does not match the grid")
    nrhs = u.size // (3 * ncell)
    rec = np.ascontiguousarray(receivers, dtype=np.float64).reshape(-1, 3)
    sa = _c128(grid.sigma_a)
    out = np.zeros((rec.shape[0], nrhs, 2, 3), np.complex128)
    _check(lib().emie_cu_receiver_fields(len(tops), _ptr(tops), _ptr(sig), grid.nz, _ptr(br), grid.nx, grid.ny,
                                         grid.hx, grid.hy, grid.x0, grid.y0, float(omega), _ptr(fp), _ptr(sa), nrhs,
                                         _ptr(u), rec.shape[0], _ptr(rec), _ptr(out)))
    return out


def kernel_output(oi: int, oj: int, hx: float, hy: float, alpha: int, beta: int, s) -> np.ndarray:
    """hankel.hpp:32 evaluated on the device (the samples the filter design uses)."""
    x = np.ascontiguousarray(np.atleast_1d(s), dtype=np.float64)
    out = np.empty_like(x)
    _check(lib().emie_cu_kernel_output(int(oi), int(oj), float(hx), float(hy), int(alpha), int(beta),
                                       _ptr(x), x.size, _ptr(out)))
    return out


class SystemOperator:
    """include/emie/cie.hpp:26-34: A = S + R1 B R2, device-resident. Holds a
    reference to its SpectralOperator (the C ABI does not own it)."""

    def __init__(self, handle, sop: SpectralOperator):
        self._h = handle
        self.b = sop

    @property
    def handle(self):
        return self._h

    def diagonals(self):
        n = self.b.nx * self.b.ny * self.b.nz
        s = np.empty(n, np.complex128)
        r1 = np.empty(n, np.float64)
        r2 = np.empty(n, np.complex128)
        _check(lib().emie_cu_system_download(self._h, _ptr(s), _ptr(r1), _ptr(r2)))
        return s, r1, r2

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.emie_cu_system_destroy(h)
            self._h = None


def contrast_coefficients(sigma_a: complex, sigma_b: complex):
    """include/emie/cie.hpp:17-24 (src/cie.cpp:9-22) -> (a, b, gamma)."""
    sa, sb = complex(sigma_a), complex(sigma_b)
    if not sb.real > 0.0:
        raise InvalidArgument("contrast coefficients: background needs Re sigma > 0")
    den = 2.0 * math.sqrt(sb.real)
    a = (sa + sb.conjugate()) / den
    b = (sa - sb) / den
    g = (sa - sb) / (sa + sb.conjugate())
    if not abs(g) < 1.0:
        raise DomainError("contrast coefficients: contraction factor reaches one")
    return a, b, g


def build_system(grid: AnomalyGrid, op: SpectralOperator) -> SystemOperator:
    """include/emie/cie.hpp:36-37 (src/cie.cpp:24-54)."""
    if grid.nx != op.nx or grid.ny != op.ny or grid.nz != op.nz:
        raise InvalidArgument("build_system: grid and operator disagree")
    sa = _c128(grid.sigma_a).reshape(-1)
    sb = _c128(grid.sigma_b)
    vol = np.array([grid.volume(iz) for iz in range(grid.nz)], dtype=np.float64)
    h = ctypes.c_void_p()
    _check(lib().emie_cu_system_create(op.handle, _ptr(sa), _ptr(sb), _ptr(vol), ctypes.byref(h)))
    return SystemOperator(h, op)


def _field_shape_check(x, ncell: int, what: str) -> int:
    n = x.numel() if _is_torch(x) else np.asarray(x).size
    if n == 0 or n % (3 * ncell) != 0:
        raise InvalidArgument(f"apply: field shape does not match {what}")
    return n // (3 * ncell)


def apply(op, v, out=None):
    """apply(SpectralOperator|SystemOperator, GridVector) (toeplitz.hpp:43,
    cie.hpp:39). v: numpy (host; copied) or torch complex128 CUDA tensor
    holding nrhs fields back to back (device-resident)."""
    L = lib()
    sop = op.b if isinstance(op, SystemOperator) else op
    ncell = sop.nx * sop.ny * sop.nz
    what = "system" if isinstance(op, SystemOperator) else "operator"
    nrhs = _field_shape_check(v, ncell, what)
    if _is_torch(v):
        import torch
        if v.dtype != torch.complex128 or not v.is_cuda or not v.is_contiguous():
            raise InvalidArgument("apply: device fields must be contiguous complex128 CUDA tensors")
        if out is None:
            out = torch.empty_like(v)
        elif (not _is_torch(out) or out.dtype != torch.complex128 or not out.is_cuda or not out.is_contiguous()
              or out.numel() != v.numel() or out.device != v.device):
            raise InvalidArgument("apply: out must be a contiguous complex128 CUDA tensor shaped like the field")
        if out.data_ptr() == v.data_ptr():
            raise InvalidArgument("apply: out may not alias the input field")
        fn = L.emie_cu_apply_system if isinstance(op, SystemOperator) else L.emie_cu_apply_spectral
        _check(fn(op.handle, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(out.data_ptr()), nrhs,
                  _stream_of()))
        return out
    import torch
    x = _c128(v)
    d_in = torch.from_numpy(x.reshape(-1)).cuda()
    d_out = torch.empty_like(d_in)
    fn = L.emie_cu_apply_system if isinstance(op, SystemOperator) else L.emie_cu_apply_spectral
    _check(fn(op.handle, ctypes.c_void_p(d_in.data_ptr()), ctypes.c_void_p(d_out.data_ptr()), nrhs,
              _stream_of()))
    return d_out.cpu().numpy().reshape(x.shape)


def apply_host(sys: SystemOperator, v: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Host buffers in/out through one C-ABI call (H2D, apply, D2H inside)."""
    x = _c128(v)
    nrhs = _field_shape_check(x, sys.b.nx * sys.b.ny * sys.b.nz, "system")
    if out is None:
        out = np.empty_like(x)
    elif (not isinstance(out, np.ndarray) or out.dtype != np.complex128 or not out.flags.c_contiguous
          or out.size != x.size):
        raise InvalidArgument("apply_host: out must be a C-contiguous complex128 array of the field's size")
    _check(lib().emie_cu_apply_system_host(sys.handle, _ptr(x), _ptr(out), nrhs, _stream_of()))
    return out


# ----------------------------------------------------------------- solve ---
@dataclass
class SolverConfig:
    """include/emie/cie.hpp:53-59. right_precond: optional flexible right
    preconditioner, a callable numpy field -> numpy field (the solve then
    runs over host callbacks); on_iteration(iteration, residual): called live
    where the reference calls it (cie.cpp:178-185, 199-201)."""
    tol: float = 1e-8
    restart: int = 40
    max_iters: int = 500
    right_precond: Optional[Callable] = None
    on_iteration: Optional[Callable] = None


@dataclass
class SolveReport:
    """include/emie/cie.hpp:43-48; status 'converged' | 'max_iterations' | 'breakdown'."""
    status: str = "max_iterations"
    iterations: int = 0
    residual: float = 0.0
    history: list = field(default_factory=list)


_STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown"}


def fgmres_system(sys: SystemOperator, rhs, config: SolverConfig = SolverConfig()):
    """fgmres (cie.hpp:71-72) with A = apply(sys, .) for nrhs right-hand
    sides in lockstep -> (x, [SolveReport]). rhs: numpy or torch CUDA tensor."""
    import torch
    ncell = sys.b.nx * sys.b.ny * sys.b.nz
    nrhs = _field_shape_check(rhs, ncell, "system")
    host = not _is_torch(rhs)
    d_rhs = torch.from_numpy(_c128(rhs).reshape(-1)).cuda() if host else rhs
    d_x = torch.empty_like(d_rhs)
    reps = (_Report * nrhs)()
    cap = max(1, config.max_iters + 1)
    hist = np.zeros((nrhs, cap), np.float64)
    hook, errs = _iteration_hook(config.on_iteration, per_rhs=nrhs > 1)
    rc = lib().emie_cu_fgmres_ex(sys.handle, ctypes.c_void_p(d_rhs.data_ptr()), ctypes.c_void_p(d_x.data_ptr()),
                                 nrhs, float(config.tol), int(config.restart), int(config.max_iters), reps,
                                 _ptr(hist), cap, hook, None, _stream_of())
    if errs:
        raise errs[0]
    _check(rc)
    out = []
    for i in range(nrhs):
        r = reps[i]
        out.append(SolveReport(_STATUS.get(r.status, "?"), r.iterations, r.residual,
                               list(hist[i, :min(r.history_len, cap)])))
    x = d_x.cpu().numpy().reshape(np.asarray(rhs).shape) if host else d_x
    return x, out


_ITER_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double)
_MAP_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                           ctypes.c_void_p)


def _iteration_hook(fn, per_rhs=False):
    """C callback for SolverConfig.on_iteration; exceptions are kept and
    re-raised after the call (no exception crosses the ABI)."""
    errs = []
    if fn is None:
        return None, errs

    def cb(_ctx, rhs, it, res):
        if errs:
            return
        try:
            fn(rhs, it, res) if per_rhs else fn(it, res)
        except BaseException as e:  # noqa: BLE001 - re-raised by the caller
            errs.append(e)
    return _ITER_FN(cb), errs


def _host_map(fn, shape, errs):
    def cb(_ctx, src, dst, n, _stream):
        try:
            x = np.ctypeslib.as_array(ctypes.cast(src, ctypes.POINTER(ctypes.c_double)), (2 * n,))
            y = np.asarray(fn(x.view(np.complex128).reshape(shape).copy()), dtype=np.complex128)
            if y.size != n:
                raise InvalidArgument("fgmres: linear map changed the field size")
            ctypes.memmove(dst, np.ascontiguousarray(y).ctypes.data, 16 * n)
            return 0
        except BaseException as e:  # noqa: BLE001 - re-raised by the caller
            errs.append(e)
            return 4
    return _MAP_FN(cb)


def fgmres(apply_a: Callable, rhs, config: SolverConfig = SolverConfig()):
    """fgmres(const LinearMap&, rhs, SolverConfig) (cie.hpp:71-72,
    cie.cpp:117-238) over a Python callable numpy field -> numpy field: the
    Krylov iteration runs on the device (emie_cu_fgmres_map), the map and the
    optional right preconditioner are called once per step on host copies.
    -> (x, SolveReport)."""
    x0 = _c128(rhs)
    n = x0.size
    if n == 0:
        raise InvalidArgument("fgmres: empty right-hand side")
    errs = []
    amap = _host_map(apply_a, x0.shape, errs)
    pmap = _host_map(config.right_precond, x0.shape, errs) if config.right_precond else None
    hook, herrs = _iteration_hook(config.on_iteration)
    x = np.zeros_like(x0)
    rep = _Report()
    cap = max(1, config.max_iters + 1)
    hist = np.zeros(cap, np.float64)
    rc = lib().emie_cu_fgmres_map(n, 1, amap, None, pmap, None, hook, None, _ptr(x0), _ptr(x), float(config.tol),
                                  int(config.restart), int(config.max_iters), ctypes.byref(rep), _ptr(hist), cap,
                                  None)
    for e in errs + herrs:
        raise e
    _check(rc)
    return x, SolveReport(_STATUS.get(rep.status, "?"), rep.iterations, rep.residual,
                          list(hist[:min(rep.history_len, cap)]))


def solve_cie(grid: AnomalyGrid, model: LayeredModel, op: SpectralOperator, rhs,
              config: SolverConfig = SolverConfig()):
    """include/emie/cie.hpp:77-80 (src/cie.cpp:240-249) -> (U, [SolveReport]).
    With config.right_precond the solve runs over host callbacks (fgmres)."""
    grid.validate(model)
    sys = build_system(grid, op)
    if config.right_precond is not None:
        x, rep = fgmres(lambda u: apply_host(sys, u), rhs, config)
        return x, [rep]
    return fgmres_system(sys, rhs, config)
