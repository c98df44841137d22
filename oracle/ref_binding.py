"""ctypes binding of the REFERENCE library built from its own sources
(oracle/_ref/libemie_ref_capi.so, see oracle/Makefile and oracle/ref_capi.cpp).

TEST INFRASTRUCTURE ONLY: used to generate and check golden fixtures and to
time the reference's CPU path. Never imported by the product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / os.environ.get("EMIE_REF_VARIANT", "_ref")  # _ref_fma: FMA-contracted build of the same sources
CAPI = REF_DIR / "libemie_ref_capi.so"
TOOL = REF_DIR / "emie_ref_tool"

_P = ctypes.POINTER(ctypes.c_double)
_lib = None


def available() -> bool:
    return CAPI.exists()


def build(quiet: bool = True) -> bool:
    """(Re)build oracle/_ref from /root/reference when that tree is present."""
    if not Path("/root/reference/proj/src").exists():
        return available()
    r = subprocess.run(["make", "-C", str(HERE), "-j8"], capture_output=quiet, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + (r.stdout or "") + (r.stderr or ""))
    return available()


def lib():
    global _lib
    if _lib is None:
        if not CAPI.exists():
            raise FileNotFoundError(f"{CAPI} missing: run `make -C oracle`")
        L = ctypes.CDLL(str(CAPI))
        L.ref_ctx_create.restype = ctypes.c_void_p
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_kernel_output.restype = ctypes.c_double
        L.ref_kernel_output.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_double]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_P)


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


class RefCase:
    """A (model, grid, omega) context inside the reference library."""

    def __init__(self, tops, sigma, breaks, nx, ny, hx, hy, omega, sigma_a=None):
        self.tops = np.ascontiguousarray(tops, np.float64)
        self.sigma = np.ascontiguousarray(sigma, np.complex128)
        self.breaks = np.ascontiguousarray(breaks, np.float64)
        self.nx, self.ny, self.nz = int(nx), int(ny), len(breaks) - 1
        self.omega = float(omega)
        sa = None if sigma_a is None else np.ascontiguousarray(sigma_a, np.complex128).reshape(-1)
        self._sa = sa
        c = lib().ref_ctx_create(len(self.tops), _dp(self.tops), _dp(self.sigma.view(np.float64)),
                                 len(self.breaks), _dp(self.breaks), self.nx, self.ny,
                                 ctypes.c_double(hx), ctypes.c_double(hy), ctypes.c_double(omega),
                                 None if sa is None else _dp(sa.view(np.float64)))
        if not c:
            raise RuntimeError(lib().ref_last_error().decode())
        self.ctx = ctypes.c_void_p(c)
        self.nent = 2 * self.nz * (2 * self.nz + 1)
        self.ncell = self.nx * self.ny * self.nz

    def __del__(self):
        if getattr(self, "ctx", None) is not None and _lib is not None:
            _lib.ref_ctx_free(self.ctx)

    def build(self):
        """assemble_operator + transform_operator + build_system -> (blocks, spectra)."""
        blocks = np.zeros((self.ny, self.nx, self.nent), np.complex128)
        dims = (ctypes.c_int * 4)()
        _check(lib().ref_build(self.ctx, _dp(blocks.view(np.float64)), None))
        _check(lib().ref_spec_dims(self.ctx, dims))
        ex, ey, qx, qy = list(dims)
        spec = np.zeros(qx * qy * self.nent, np.complex128)
        _check(lib().ref_build(self.ctx, None, _dp(spec.view(np.float64))))
        return blocks, spec, (ex, ey, qx, qy)

    def set_operator(self, blocks):
        b = np.ascontiguousarray(blocks, np.complex128)
        _check(lib().ref_set_operator(self.ctx, _dp(b.view(np.float64))))

    def apply(self, which: str, v):
        w = {"spectral": 0, "system": 1, "dense": 2}[which]
        x = np.ascontiguousarray(v, np.complex128).reshape(-1)
        out = np.zeros_like(x)
        _check(lib().ref_apply(self.ctx, w, _dp(x.view(np.float64)), _dp(out.view(np.float64))))
        return out

    def diagonals(self):
        s = np.zeros(self.ncell, np.complex128)
        r1 = np.zeros(self.ncell, np.float64)
        r2 = np.zeros(self.ncell, np.complex128)
        _check(lib().ref_system_diagonals(self.ctx, _dp(s.view(np.float64)), _dp(r1),
                                          _dp(r2.view(np.float64))))
        return s, r1, r2

    def solve(self, rhs, tol, restart=40, max_iters=500):
        b = np.ascontiguousarray(rhs, np.complex128).reshape(-1)
        x = np.zeros_like(b)
        rep = np.zeros(3)
        hist = np.zeros(max_iters + 1)
        hl = ctypes.c_int(0)
        _check(lib().ref_solve(self.ctx, _dp(b.view(np.float64)), ctypes.c_double(tol), restart,
                               max_iters, _dp(x.view(np.float64)), _dp(rep), _dp(hist),
                               len(hist), ctypes.byref(hl)))
        status = {0: "converged", 1: "max_iterations", 2: "breakdown"}[int(rep[0])]
        return x, {"status": status, "iterations": int(rep[1]), "residual": float(rep[2]),
                   "history": hist[:hl.value].tolist()}

    def block(self, oi, oj):
        out = np.zeros(self.nent, np.complex128)
        _check(lib().ref_assemble_block(self.ctx, int(oi), int(oj), _dp(out.view(np.float64))))
        return out

    def block_weights(self, oi, oj, w, lam, r=0.0):
        """assemble_block's accumulation with given filter weights w (6, nw), lam (nw)
        (r > 0: that reference distance instead of pair_geometry's)."""
        w = np.ascontiguousarray(w, np.float64)
        lam = np.ascontiguousarray(lam, np.float64)
        out = np.zeros(self.nent, np.complex128)
        _check(lib().ref_assemble_block_weights(self.ctx, int(oi), int(oj), _dp(w), _dp(lam), len(lam),
                                                _dp(out.view(np.float64)), ctypes.c_double(r)))
        return out

    def vfunctions(self, lam):
        """v_functions of every (n, m) pair at lam -> (5, nz, nz)."""
        out = np.zeros(5 * self.nz * self.nz, np.complex128)
        _check(lib().ref_vfunctions(self.ctx, ctypes.c_double(lam), _dp(out.view(np.float64))))
        return out.reshape(5, self.nz, self.nz)

    def block_full(self, oi, oj):
        out = np.zeros(9 * self.nz * self.nz, np.complex128)
        _check(lib().ref_assemble_block_full(self.ctx, int(oi), int(oj), _dp(out.view(np.float64))))
        return out.reshape(9, self.nz, self.nz)


def design_weights(oi, oj, hx, hy, alpha, beta):
    w = np.zeros(451)
    lam = np.zeros(451)
    _check(lib().ref_design_weights(oi, oj, ctypes.c_double(hx), ctypes.c_double(hy), alpha, beta,
                                    _dp(w), _dp(lam)))
    return w, lam


def moment_tables(tops, sigma, breaks, omega, lam):
    tops = np.ascontiguousarray(tops, np.float64)
    sig = np.ascontiguousarray(sigma, np.complex128)
    br = np.ascontiguousarray(breaks, np.float64)
    nz = len(br) - 1
    t = np.zeros(12 * nz * nz, np.complex128)
    _check(lib().ref_moment_tables(len(tops), _dp(tops), _dp(sig.view(np.float64)), len(br), _dp(br),
                                   ctypes.c_double(omega), ctypes.c_double(lam), _dp(t.view(np.float64))))
    return t.reshape(2, 6, nz, nz)


def write_case(path, tops, sigma, breaks, nx, ny, hx, hy, omega, sigma_a=None, vecs=(), rhs=(),
               tol=1e-8, restart=40, max_iters=500):
    """Binary case file read by oracle/_ref/emie_ref_tool (oracle/ref_tool.cpp)."""
    with open(path, "wb") as f:
        f.write(b"EMCASE1\0")
        f.write(np.int32(len(tops)).tobytes())
        f.write(np.asarray(tops, np.float64).tobytes())
        f.write(np.asarray(sigma, np.complex128).tobytes())
        f.write(np.int32(len(breaks)).tobytes())
        f.write(np.asarray(breaks, np.float64).tobytes())
        f.write(np.int32(nx).tobytes() + np.int32(ny).tobytes())
        f.write(np.asarray([hx, hy, 0.0, 0.0, omega], np.float64).tobytes())
        if sigma_a is None:
            f.write(np.int32(0).tobytes())
        else:
            f.write(np.int32(1).tobytes())
            f.write(np.asarray(sigma_a, np.complex128).reshape(-1).tobytes())
        f.write(np.int32(len(vecs)).tobytes())
        for v in vecs:
            f.write(np.asarray(v, np.complex128).reshape(-1).tobytes())
        f.write(np.int32(len(rhs)).tobytes())
        for v in rhs:
            f.write(np.asarray(v, np.complex128).reshape(-1).tobytes())
        f.write(np.float64(tol).tobytes() + np.int32(restart).tobytes() + np.int32(max_iters).tobytes())


def run_tool(*args, threads=None, timeout=3600):
    env = dict(os.environ)
    if threads:
        env["OMP_NUM_THREADS"] = str(threads)
    r = subprocess.run([str(TOOL)] + [str(a) for a in args], capture_output=True, text=True,
                       env=env, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"emie_ref_tool failed: {r.stderr}")
    return r.stdout
