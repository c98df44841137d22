"""Forward modelling pipeline (the reference has only
placeholders, src/pipeline.cpp:1 and tools/emie_main.cpp:1).

Per period: Green's build on the device (or an EMG1 snapshot from the cache,
greens.cpp:373-446 format), spectra, both plane-wave polarisations solved in
lockstep on the device, anomalous receiver fields on the device (paper Eq.
APR_lab), normal fields of the 1-D background, MT impedances.

Config (YAML, SPEC.md External Interfaces):

    layers:            # each layer below its top interface; the last is the lower halfspace
      - {top_depth_m: 0.0, conductivity_S_per_m: 0.01}
      - {top_depth_m: 1000.0, conductivity_S_per_m: 0.001}
      - {top_depth_m: 11000.0, conductivity_S_per_m: 0.1}
    air_S_per_m: 0.0   # optional (floored to 1e-9, layered.cpp:47-51)
    grid: {origin_m: [0, 0], nx: 16, ny: 16, hx_m: 500, hy_m: 500, z_breaks_m: [0, 250, ...]}
    blocks:            # cells take the conductivity of the last block covering their centre
      - {corner1_m: [x, y, z], corner2_m: [x, y, z], conductivity_S_per_m: 1.0}
    periods_s: [10.0]
    receivers: [[x, y, z], ...]   # or {x_m: [start, stop, n], y_m: [start, stop, n], z_m: 0.0}
    solver: {tol: 1.0e-6, restart: 40, max_iter: 500}
    cache_dir: /tmp/emie_cache    # optional

Outputs: one CSV per period (SPEC.md header, 9 significant digits) and a
convergence log (iter,relative_residual) per period and polarisation.
"""
from __future__ import annotations

import hashlib
import json
import math
import struct
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np

from . import normal_field as NF

MU0 = 1.2566370614359172e-06
CSV_HEADER = ("x_m,y_m,period_s,re_Zxx,im_Zxx,re_Zxy,im_Zxy,re_Zyx,im_Zyx,re_Zyy,im_Zyy,"
              "rho_xy_ohmm,phi_xy_deg,rho_yx_ohmm,phi_yx_deg")


class ConfigError(ValueError):
    """A validation failure of the forward config (structured diagnostics)."""


# ------------------------------------------------------------ responses ----
@dataclass
class ImpedanceResponse:
    """SPEC.md ImpedanceResponse: Z (2x2, Ohm), apparent resistivities and
    phases (degrees, e^{+i w t} MT convention, in (-180, 180])."""
    position: tuple
    period: float
    Z: np.ndarray
    rho_xy: float
    rho_yx: float
    phi_xy: float
    phi_yx: float


def _phase(z: complex) -> float:
    p = math.degrees(math.atan2(-z.imag, z.real))  # arg(conj Z)
    return 180.0 if p == -180.0 else p


def mt_responses(E, H, receivers, omega: float) -> List[ImpedanceResponse]:
    """mt_responses: E, H (nrec, 2 polarisations, 3) total fields;
    Z solves [Ex Ey] = Z [Hx Hy] across the polarisations (2x2 per receiver)."""
    E = np.asarray(E)
    H = np.asarray(H)
    out = []
    T = 2 * math.pi / omega
    for i, pos in enumerate(np.asarray(receivers, dtype=np.float64).reshape(-1, 3)):
        Em = E[i, :, :2].T  # columns: polarisations; rows: x, y
        Hm = H[i, :, :2].T
        det = Hm[0, 0] * Hm[1, 1] - Hm[0, 1] * Hm[1, 0]
        scale = max(abs(Hm).max() ** 2, 1e-300)
        if abs(det) <= 1e-12 * scale:
            raise ArithmeticError(f"mt_responses: singular magnetic field matrix at receiver {i}")
        Z = Em @ np.linalg.inv(Hm)
        rho = lambda z: abs(z) ** 2 / (omega * MU0)  # noqa: E731
        out.append(ImpedanceResponse(tuple(pos), T, Z, rho(Z[0, 1]), rho(Z[1, 0]), _phase(Z[0, 1]),
                                     _phase(Z[1, 0])))
    return out


def csv_rows(responses: List[ImpedanceResponse]) -> str:
    f = lambda v: f"{v:.8e}"  # noqa: E731  (9 significant digits)
    lines = [CSV_HEADER]
    for r in responses:
        z = r.Z
        vals = [r.position[0], r.position[1], r.period, z[0, 0].real, z[0, 0].imag, z[0, 1].real, z[0, 1].imag,
                z[1, 0].real, z[1, 0].imag, z[1, 1].real, z[1, 1].imag, r.rho_xy, r.phi_xy, r.rho_yx, r.phi_yx]
        lines.append(",".join(f(v) for v in vals))
    return "\n".join(lines) + "\n"


# --------------------------------------------------------------- config ----
@dataclass
class ForwardConfig:
    tops: list
    sigma: list  # complex; [0] = air
    origin: tuple
    nx: int
    ny: int
    hx: float
    hy: float
    breaks: list
    blocks: list = field(default_factory=list)
    periods: list = field(default_factory=list)
    receivers: np.ndarray = None
    tol: float = 1e-6
    restart: int = 40
    max_iter: int = 500
    cache_dir: Optional[str] = None

    def key(self, period: float) -> str:
        """Cache key of a period's operator: everything the Green's build reads."""
        d = json.dumps([self.tops, [[complex(s).real, complex(s).imag] for s in self.sigma], self.nx, self.ny,
                        self.hx, self.hy, self.breaks, period], sort_keys=True)
        return hashlib.sha256(d.encode()).hexdigest()[:24]


def _need(d, k, where):
    if k not in d:
        raise ConfigError(f"config: missing '{k}' in {where}")
    return d[k]


def parse_config(d: dict) -> ForwardConfig:
    layers = _need(d, "layers", "the config")
    if not layers:
        raise ConfigError("config: 'layers' is empty")
    tops = [float(_need(l, "top_depth_m", "a layer")) for l in layers]
    sig = [complex(float(d.get("air_S_per_m", 0.0)))] + [complex(float(_need(l, "conductivity_S_per_m", "a layer")))
                                                         for l in layers]
    for a, b in zip(tops, tops[1:]):
        if not b > a:
            raise ConfigError("config: layer tops must increase")
    if any(s.real < 0 for s in sig):
        raise ConfigError("config: negative conductivity")
    g = _need(d, "grid", "the config")
    origin = tuple(float(v) for v in g.get("origin_m", [0.0, 0.0]))
    nx, ny = int(_need(g, "nx", "grid")), int(_need(g, "ny", "grid"))
    hx, hy = float(_need(g, "hx_m", "grid")), float(_need(g, "hy_m", "grid"))
    breaks = [float(z) for z in _need(g, "z_breaks_m", "grid")]
    if "nz" in g and int(g["nz"]) != len(breaks) - 1:
        raise ConfigError("config: grid.nz disagrees with z_breaks_m")
    if nx < 1 or ny < 1 or len(breaks) < 2 or not (hx > 0 and hy > 0):
        raise ConfigError("config: empty or degenerate grid")
    blocks = []
    for b in d.get("blocks", []) or []:
        c1 = [float(v) for v in _need(b, "corner1_m", "a block")]
        c2 = [float(v) for v in _need(b, "corner2_m", "a block")]
        s = float(_need(b, "conductivity_S_per_m", "a block"))
        if s < 0:
            raise ConfigError("config: negative block conductivity")
        blocks.append((np.minimum(c1, c2), np.maximum(c1, c2), s))
    periods = [float(p) for p in _need(d, "periods_s", "the config")]
    if not periods or any(not p > 0 for p in periods):
        raise ConfigError("config: periods must be positive")
    rec = d.get("receivers")
    if isinstance(rec, dict):
        xs = np.linspace(*[float(v) for v in rec["x_m"][:2]], int(rec["x_m"][2]))
        ys = np.linspace(*[float(v) for v in rec["y_m"][:2]], int(rec["y_m"][2]))
        z = float(rec.get("z_m", 0.0))
        recs = np.array([[x, y, z] for y in ys for x in xs], dtype=np.float64)
    else:
        recs = np.asarray(rec if rec is not None else [], dtype=np.float64).reshape(-1, 3)
    s = d.get("solver", {}) or {}
    return ForwardConfig(tops, sig, origin, nx, ny, hx, hy, breaks, blocks, periods, recs,
                         float(s.get("tol", 1e-6)), int(s.get("restart", 40)), int(s.get("max_iter", 500)),
                         d.get("cache_dir"))


def load_config(path) -> ForwardConfig:
    import yaml
    with open(path) as f:
        return parse_config(yaml.safe_load(f))


def build_model(cfg: ForwardConfig):
    """LayeredModel + AnomalyGrid with the block conductivities (last covering
    block wins, background elsewhere); raises the library's errors for grids
    crossing layers or intervals in the air."""
    import paper_1512_06126_b200 as emie
    model = emie.LayeredModel(list(cfg.tops), list(cfg.sigma))
    grid = emie.make_grid(model, list(cfg.breaks), cfg.nx, cfg.ny, cfg.hx, cfg.hy, cfg.origin[0], cfg.origin[1])
    if cfg.blocks:
        xc = cfg.origin[0] + (np.arange(cfg.nx) + 0.5) * cfg.hx
        yc = cfg.origin[1] + (np.arange(cfg.ny) + 0.5) * cfg.hy
        zc = 0.5 * (np.asarray(cfg.breaks[:-1]) + np.asarray(cfg.breaks[1:]))
        Z, Y, X = np.meshgrid(zc, yc, xc, indexing="ij")
        for lo, hi, s in cfg.blocks:
            inside = (X >= lo[0]) & (X <= hi[0]) & (Y >= lo[1]) & (Y <= hi[1]) & (Z >= lo[2]) & (Z <= hi[2])
            grid.sigma_a[inside] = s
    return model, grid


# --------------------------------------------------------- EMG1 cache ----
def save_operator(path, blocks: np.ndarray, nx: int, ny: int, nz: int, omega: float) -> None:
    """EMG1 snapshot (greens.cpp:373-446 format): magic, dims, omega, then per
    block the six components each as (count, complex data)."""
    nt, nf = nz * (nz + 1) // 2, nz * nz
    b = np.ascontiguousarray(blocks, np.complex128).reshape(ny * nx, -1)
    with open(path, "wb") as f:
        f.write(struct.pack("<I3id", 0x454D4731, nx, ny, nz, omega))
        for blk in b:
            o = 0
            for n in (nt, nt, nt, nt, nf, nf):
                f.write(struct.pack("<Q", n))
                f.write(blk[o:o + n].tobytes())
                o += n


def load_operator(path, nx: int, ny: int, nz: int):
    """-> (blocks (ny, nx, nent), omega) or None for an absent/foreign/truncated file."""
    p = Path(path)
    if not p.exists():
        return None
    data = p.read_bytes()
    if len(data) < 24:
        return None
    magic, dx, dy, dz, omega = struct.unpack_from("<I3id", data, 0)
    if magic != 0x454D4731 or (dx, dy, dz) != (nx, ny, nz):
        return None
    nt, nf = nz * (nz + 1) // 2, nz * nz
    out = np.zeros((ny * nx, 2 * nz * (2 * nz + 1)), np.complex128)
    pos = 24
    for i in range(ny * nx):
        o = 0
        for n in (nt, nt, nt, nt, nf, nf):
            if pos + 8 > len(data):
                return None
            (cnt,) = struct.unpack_from("<Q", data, pos)
            pos += 8
            if cnt != n or pos + 16 * n > len(data):
                return None
            out[i, o:o + n] = np.frombuffer(data, np.complex128, n, pos)
            pos += 16 * n
            o += n
    return out.reshape(ny, nx, -1), omega


# --------------------------------------------------------------- forward ----
def reconstruct_fields(grid, model, omega: float, U, receivers):
    """reconstruct_fields: total E and H at the receivers for the two
    polarisation solutions U (2, 3N) -> E, H each (nrec, 2, 3)."""
    import paper_1512_06126_b200 as emie
    anom = emie.receiver_fields(grid, model, omega, U, receivers)  # (nrec, 2, 2, 3)
    En, Hn = NF.normal_fields(model.tops, model.sigma, omega, receivers)
    return En + anom[:, :, 0], Hn + anom[:, :, 1]


def run_forward(cfg: ForwardConfig, out_dir, use_cache: bool = True, log=print) -> List[Path]:
    """run_forward: per period filters -> assembly (or cache load) ->
    spectra -> two-polarisation solve -> receiver fields -> responses CSV."""
    import paper_1512_06126_b200 as emie
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    model, grid = build_model(cfg)
    if len(cfg.receivers) == 0:
        raise ConfigError("config: no receivers")
    written = []
    for period in cfg.periods:
        omega = 2 * math.pi / period
        cache = Path(cfg.cache_dir) / f"emg1_{cfg.key(period)}.bin" if (cfg.cache_dir and use_cache) else None
        sop, src = None, "device Green's build"
        if cache is not None:
            got = load_operator(cache, cfg.nx, cfg.ny, grid.nz)
            if got is not None:
                sop = emie.transform_operator(got[0], cfg.nx, cfg.ny, grid.nz, got[1])
                src = f"cache {cache.name}"
        if sop is None:
            sop = emie.assemble_operator(grid, model, omega, keep_blocks=cache is not None)
            if cache is not None:
                cache.parent.mkdir(parents=True, exist_ok=True)
                save_operator(cache, sop.blocks(), cfg.nx, cfg.ny, grid.nz, omega)
        rhs = np.stack([NF.build_rhs(model.tops, model.sigma, grid.breaks, cfg.nx, cfg.ny, omega, p) for p in "xy"])
        hist = []
        conf = emie.SolverConfig(tol=cfg.tol, restart=cfg.restart, max_iters=cfg.max_iter,
                                 on_iteration=lambda r, it, res: hist.append((r, it, res)))
        U, reps = emie.fgmres_system(emie.build_system(grid, sop), rhs, conf)
        for k, rep in enumerate(reps):
            if rep.status != "converged":
                log(f"period {period:g} s, polarisation {'xy'[k]}: {rep.status} after {rep.iterations} "
                    f"iterations (residual {rep.residual:.3e})")
        E, H = reconstruct_fields(grid, model, omega, U, cfg.receivers)
        res = mt_responses(E, H, cfg.receivers, omega)
        f = out / f"responses_T{period:.9g}s.csv"
        f.write_text(csv_rows(res))
        conv = out / f"convergence_T{period:.9g}s.log"
        conv.write_text("".join(f"{'xy'[r]},{it},{v:.9e}\n" for r, it, v in hist))
        log(f"period {period:g} s: operator from {src}; iterations {[r.iterations for r in reps]}; wrote {f.name}")
        written.append(f)
    return written


def responses_1d(cfg: ForwardConfig, out_dir) -> List[Path]:
    """responses1d (SPEC.md CLI): background-only MT responses at the
    receivers (the normal field; no anomaly)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = []
    for period in cfg.periods:
        omega = 2 * math.pi / period
        E, H = NF.normal_fields(cfg.tops, cfg.sigma, omega, cfg.receivers)
        f = out / f"responses1d_T{period:.9g}s.csv"
        f.write_text(csv_rows(mt_responses(E, H, cfg.receivers, omega)))
        written.append(f)
    return written
