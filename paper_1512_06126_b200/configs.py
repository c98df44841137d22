"""The five BASELINE.json configurations as seeded synthetic models.

BASELINE.json names no public dataset; every conductivity field here is
generated from a fixed seed (numpy PCG64, seed 20151218 + cfg) so the
reference oracle and the B200 path see identical bytes. Decisions the
survey left open are pinned here:
  - configs 3-5: lower halfspace sigma = 1 S/m;
  - config 2: white noise smoothed by a separable Gaussian (sigma 3 cells
    laterally, 1.5 vertically, reflecting edges), standardised exactly to
    mean -2 / sd 0.7 in log10 sigma;
  - config 3: log10 sigma ~ U[-4, 1] per 8x8x4-cell block plus 8 boxes of
    side U{4..16} cells with log10 sigma ~ U[0, 1];
  - config 4: log10 sigma ~ U[-4, 1] per 8x8x4-cell block.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CFG1_MODEL = ([0.0, 1000.0, 11000.0], [0.0, 0.01, 0.001, 0.1])
CFG3_MODEL = ([0.0, 500.0, 2500.0, 7500.0, 17500.0, 37500.0],
              [0.0, 1e-3, 10 ** -2.25, 10 ** -1.5, 10 ** -0.75, 1.0, 1.0])


@dataclass
class Config:
    name: str
    tops: list
    sigma: list
    breaks: list
    nx: int
    ny: int
    hx: float
    hy: float
    freqs: list
    sigma_a: np.ndarray  # (nz, ny, nx) complex128

    @property
    def nz(self):
        return len(self.breaks) - 1

    @property
    def omega(self):
        return 2.0 * np.pi * self.freqs[0]

    def cells(self):
        return self.nx * self.ny * self.nz


def _blocky(rng, nz, ny, nx, bz, by, bx, lo, hi):
    gz, gy, gx = -(-nz // bz), -(-ny // by), -(-nx // bx)
    vals = rng.uniform(lo, hi, size=(gz, gy, gx))
    return np.repeat(np.repeat(np.repeat(vals, bz, 0), by, 1), bx, 2)[:nz, :ny, :nx]


def config(k: int) -> Config:
    rng = np.random.default_rng(20151218 + k)
    if k == 1:
        tops, sig = CFG1_MODEL
        breaks = list(np.arange(0.0, 2000.0 + 1e-9, 250.0))
        nx = ny = 16
        lg = _blocky(rng, 8, ny, nx, 2, 4, 4, -3.0, 0.0)
        return Config("cfg1", tops, sig, breaks, nx, ny, 500.0, 500.0, [0.1], (10.0 ** lg).astype(np.complex128))
    if k == 2:
        from scipy.ndimage import gaussian_filter
        tops, sig = CFG1_MODEL
        breaks = list(np.arange(0.0, 2000.0 + 1e-9, 125.0))
        nx = ny = 64
        w = rng.standard_normal((16, ny, nx))
        s = gaussian_filter(w, sigma=(1.5, 3.0, 3.0), mode="reflect")
        lg = -2.0 + 0.7 * (s - s.mean()) / s.std()
        return Config("cfg2", tops, sig, breaks, nx, ny, 250.0, 250.0, [0.01, 0.1, 1.0],
                      (10.0 ** lg).astype(np.complex128))
    if k in (3, 5):
        tops, sig = CFG3_MODEL
        breaks = list(np.arange(0.0, 3200.0 + 1e-9, 100.0))
        nx = ny = 128
        nz = 32
        rng = np.random.default_rng(20151218 + 3)
        lg = _blocky(rng, nz, ny, nx, 4, 8, 8, -4.0, 1.0)
        for _ in range(8):
            sx, sy, sz = rng.integers(4, 17, size=3)
            x0, y0, z0 = rng.integers(0, nx - sx + 1), rng.integers(0, ny - sy + 1), rng.integers(0, nz - sz + 1)
            lg[z0:z0 + sz, y0:y0 + sy, x0:x0 + sx] = rng.uniform(0.0, 1.0)
        freqs = [1.0] if k == 3 else list(np.logspace(-3, 2, 32))
        return Config(f"cfg{k}", tops, sig, breaks, nx, ny, 200.0, 200.0, freqs,
                      (10.0 ** lg).astype(np.complex128))
    if k == 4:
        tops, sig = CFG3_MODEL
        breaks = list(np.arange(0.0, 3200.0 + 1e-9, 50.0))
        nx = ny = 256
        lg = _blocky(rng, 64, ny, nx, 4, 8, 8, -4.0, 1.0)
        return Config("cfg4", tops, sig, breaks, nx, ny, 100.0, 100.0, [0.1], (10.0 ** lg).astype(np.complex128))
    raise ValueError(f"no config {k}")
