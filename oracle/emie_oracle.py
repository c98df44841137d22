"""CPU restatement (numpy) of the reference's hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 implementation. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it; the
product library (paper_1512_06126_b200) never does.

Every function cites the reference file:line it restates (paths relative to
/root/reference/proj). It is pinned against the reference itself, compiled
from its own sources by oracle/Makefile (oracle/_ref), through the golden
fixtures in tests/golden/ (tests/test_oracle_pins.py).

Conventions: complex128 everywhere; GridVector layout
((c*nz + iz)*ny + iy)*nx + ix (include/emie/types.hpp:14-30).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MU0 = 1.2566370614359172e-06  # include/emie/types.hpp:11
PI = 3.141592653589793238462643383279502884
SIGMA_FLOOR = 1e-9  # include/emie/layered.hpp:32
PARITY_X = (1, 1, 1, -1, -1, 1)  # src/toeplitz.cpp:59
PARITY_Y = (1, 1, 1, -1, 1, -1)  # src/toeplitz.cpp:60


# ---------------------------------------------------------------- models ---
@dataclass
class LayeredModel:
    """include/emie/layered.hpp:15-33; src/layered.cpp:32-65."""
    tops: list
    sigma: list  # complex, len(tops)+1

    @property
    def L(self):
        return len(self.tops)

    def layer_of(self, z):  # layered.cpp:32-36 (points on an interface go below)
        import bisect
        return bisect.bisect_right(self.tops, z)

    def top_of(self, m):  # layered.cpp:38
        return self.tops[0] if m == 0 else self.tops[m - 1]

    def bottom_of(self, m):  # layered.cpp:40-43
        return self.tops[-1] if m == self.L else self.tops[m]

    def thickness(self, m):  # layered.cpp:45
        return self.bottom_of(m) - self.top_of(m)

    def sigma_floored(self, m):  # layered.cpp:47-51
        s = complex(self.sigma[m])
        if s.real < SIGMA_FLOOR:
            s = complex(SIGMA_FLOOR, s.imag)
        return s

    def validate(self):  # layered.cpp:53-65
        if not self.tops:
            raise ValueError("layered model needs at least one interface")
        if len(self.sigma) != len(self.tops) + 1:
            raise ValueError("layered model: sigma count must be tops count + 1")
        for a, b in zip(self.tops, self.tops[1:]):
            if not a < b:
                raise ValueError("layered model: interface depths must increase")


def partition_layers(model: LayeredModel, breaks):
    """VerticalPartition::create (src/layered.cpp:191-208)."""
    if len(breaks) < 2:
        raise ValueError("vertical partition needs at least one interval")
    L = model.L
    layer = []
    for i in range(len(breaks) - 1):
        if not breaks[i] < breaks[i + 1]:
            raise ValueError("vertical partition: breaks must increase")
        m = model.layer_of(breaks[i])
        slack = 1e-7 * (1.0 + abs(breaks[i + 1]))
        if m < L and breaks[i + 1] > model.bottom_of(m) + slack:
            raise ValueError("vertical partition: interval straddles a layer interface")
        layer.append(m)
    return layer


@dataclass
class Grid:
    """AnomalyGrid / make_grid (include/emie/greens.hpp:22-45, src/greens.cpp:18-57)."""
    model: LayeredModel
    breaks: list
    nx: int
    ny: int
    hx: float
    hy: float
    layer: list = field(default_factory=list)
    sigma_b: np.ndarray = None
    sigma_a: np.ndarray = None  # (nz, ny, nx) complex

    @property
    def nz(self):
        return len(self.breaks) - 1

    def dz(self, iz):
        return self.breaks[iz + 1] - self.breaks[iz]

    def volume(self, iz):  # greens.hpp:35
        return self.hx * self.hy * self.dz(iz)


def make_grid(model, breaks, nx, ny, hx, hy, sigma_a=None):
    """src/greens.cpp:37-57 plus validate (18-35)."""
    model.validate()
    if nx <= 0 or ny <= 0:
        raise ValueError("grid: empty dimensions")
    if not (hx > 0 and hy > 0):
        raise ValueError("grid: cell sizes must be positive")
    layer = partition_layers(model, list(breaks))
    g = Grid(model, list(breaks), nx, ny, hx, hy, layer)
    g.sigma_b = np.array([model.sigma_floored(m) for m in layer], dtype=np.complex128)
    if sigma_a is None:
        sigma_a = np.broadcast_to(g.sigma_b[:, None, None], (g.nz, ny, nx)).copy()
    g.sigma_a = np.asarray(sigma_a, dtype=np.complex128).reshape(g.nz, ny, nx)
    if np.any(~(g.sigma_a.real >= 0)):
        raise ValueError("grid: cell conductivity with negative real part")
    for m in layer:
        if not model.sigma[m].real > 0:
            raise ValueError("grid: interval in a non-conducting layer")
    return g


# ---------------------------------------------------- hankel filters -------
FILTER_STEP, FILTER_SHIFT, FILTER_HALF, FILTER_N1, FILTER_N2 = 0.2, 0.0964, 512, -250, 200
AB6 = ((0, 0), (2, 0), (0, 2), (1, 1), (1, 0), (0, 1))  # src/greens.cpp:137


def pair_geometry(oi, oj, hx, hy):
    """src/hankel.cpp:80-91 -> (r, p, q, phi)."""
    ax = oj * hx - 0.5 * hx
    ay = oi * hy - 0.5 * hy
    r = math.hypot(ax, ay)
    return r, hx / r, hy / r, math.atan2(ay, ax)


def design_input(lam):
    """src/hankel.cpp:93-99 (vectorised)."""
    lam = np.asarray(lam, dtype=np.float64)
    l2 = lam * lam
    with np.errstate(over="ignore", invalid="ignore"):
        v = 8.0 * np.exp(-l2) * lam * ((l2 - 4.0) * l2 + 2.0)
    return np.where(lam > 38.0, 0.0, v)


def _erf(x):
    from scipy.special import erf
    return erf(x)


def _erfc(x):
    from scipy.special import erfc
    return erfc(x)


def _ediff(a, b):
    """src/hankel.cpp:22-26 (vectorised)."""
    both_pos = (a > 1.0) & (b > 1.0)
    both_neg = (a < -1.0) & (b < -1.0)
    out = _erf(0.5 * b) - _erf(0.5 * a)
    out = np.where(both_pos, _erfc(0.5 * a) - _erfc(0.5 * b), out)
    out = np.where(both_neg, _erfc(-0.5 * b) - _erfc(-0.5 * a), out)
    return out


def _axis_stencil(alpha, d, h):
    """src/hankel.cpp:35-71 (vectorised over d, h) -> (out0, out1, out2)."""
    sp = 1.7724538509055160273
    wp, w0, wm = d + h, d, d - h
    gp, g0, gm = np.exp(-0.25 * wp * wp), np.exp(-0.25 * w0 * w0), np.exp(-0.25 * wm * wm)
    gs = gp - 2.0 * g0 + gm
    ep = _ediff(w0, wp)
    em = _ediff(wm, w0)
    if alpha == 0:
        lin = wp * ep - wm * em
        w2s = wp * wp * gp - 2.0 * w0 * w0 * g0 + wm * wm * gm
        return (sp * lin + 2.0 * gs, 2.0 * sp * lin + 8.0 * gs,
                12.0 * sp * lin + 4.0 * w2s + 64.0 * gs)
    if alpha == 1:
        es = ep - em
        wg = wp * gp - 2.0 * w0 * g0 + wm * gm
        w3g = wp * wp * wp * gp - 2.0 * w0 * w0 * w0 * g0 + wm * wm * wm * gm
        return (sp * es, 2.0 * sp * es - 2.0 * wg, 12.0 * sp * es - 2.0 * w3g - 12.0 * wg)
    if alpha == 2:
        return (gs, wp * wp * gp - 2.0 * w0 * w0 * g0 + wm * wm * gm,
                wp ** 4 * gp - 2.0 * w0 ** 4 * g0 + wm ** 4 * gm)
    raise ValueError("axis_stencil: derivative order")


def kernel_output(geom, alpha, beta, s):
    """src/hankel.cpp:101-113 (vectorised over s)."""
    if alpha < 0 or beta < 0 or alpha > 2 or beta > 2 or alpha + beta > 2:
        raise ValueError("kernel orders: need alpha, beta >= 0 and alpha + beta <= 2")
    _, p, q, phi = geom
    s = np.asarray(s, dtype=np.float64)
    r = np.exp(s)
    hx, hy = p * r, q * r
    dx = r * math.cos(phi) + 0.5 * hx
    dy = r * math.sin(phi) + 0.5 * hy
    ax = _axis_stencil(alpha, dx, hx)
    ay = _axis_stencil(beta, dy, hy)
    comb = 0.25 * (ax[2] * ay[0] + 2.0 * ax[1] * ay[1] + ax[0] * ay[2])
    with np.errstate(over="ignore", invalid="ignore"):
        out = np.exp(-(3 - alpha - beta) * s) * comb
    return np.where(comb == 0.0, 0.0, out)


def _alt_signs(n, half):
    j = np.arange(n)
    return np.where((j + half) % 2 == 0, 1.0, -1.0)


def filter_denominator(half=FILTER_HALF, step=FILTER_STEP):
    """FilterDesigner ctor (src/hankel.cpp:204-232): input spectrum and floor."""
    n = 2 * half
    m = np.arange(n) - half
    den = np.fft.fft(_alt_signs(n, half) * design_input(np.exp(-m * step)))
    return den, 1e-12 * np.max(np.abs(den))


def design_weights(geom, alpha, beta, half=FILTER_HALF, step=FILTER_STEP,
                   shift=FILTER_SHIFT, n1=FILTER_N1, n2=FILTER_N2, den=None):
    """FilterDesigner::design (src/hankel.cpp:239-281) -> (w, lam)."""
    n = 2 * half
    if den is None:
        den, floor = filter_denominator(half, step)
    else:
        den, floor = den
    m = np.arange(n) - half
    u = _alt_signs(n, half) * kernel_output(geom, alpha, beta, m * step + shift)
    spec = np.fft.fft(u)
    if np.any(np.abs(den) < floor):
        raise RuntimeError("filter design: input spectrum vanishes at a used mode")
    buf = np.fft.ifft(spec / den) * n  # unnormalised backward transform
    remax, immax = np.max(np.abs(buf.real)), np.max(np.abs(buf.imag))
    if immax > 1e-10 * remax:
        raise RuntimeError("filter design: weights have a non-real residue")
    mm = np.arange(n1, n2 + 1)
    j = np.mod(mm, n)
    sign = np.where(mm % 2 != 0, -1.0, 1.0)
    w = sign * buf.real[j] / n
    lam = np.exp(mm * step + shift)
    return w, lam


# ------------------------------------------------------- layered kernels ---
def _cexpm1(x):
    """exp(x) - 1 without cancellation (src/layered.cpp:19-25)."""
    em = np.expm1(x.real)
    s = np.sin(0.5 * x.imag)
    return (em * np.cos(x.imag) - 2.0 * s * s) + 1j * ((em + 1.0) * np.sin(x.imag))


@dataclass
class LayerState:
    """SpectralLayerState, vectorised over lambda: arrays (nlam, L+1)."""
    sig: np.ndarray
    eta: np.ndarray
    p: np.ndarray
    q: np.ndarray
    one_p: np.ndarray
    one_q: np.ndarray
    e2l: np.ndarray
    em1_2l: np.ndarray
    diag_a: np.ndarray


def spectral_state(model: LayeredModel, omega, lam, cond):
    """build_spectral_state (src/layered.cpp:67-129), vectorised over lam."""
    lam = np.atleast_1d(np.asarray(lam, dtype=np.float64))
    L = model.L
    nl = lam.size
    sig = np.array([model.sigma_floored(m) for m in range(L + 1)], dtype=np.complex128)
    eta2 = (lam * lam)[:, None] + 0j - (1j * omega * MU0) * sig[None, :]
    eta = np.sqrt(eta2)
    eta = np.where(eta.real < 0.0, -eta, eta)
    e2l = np.ones((nl, L + 1), np.complex128)
    em1 = np.zeros((nl, L + 1), np.complex128)
    for m in range(1, L):
        x = _cexpm1(-2.0 * eta[:, m] * model.thickness(m))
        e2l[:, m] = 1.0 + x
        em1[:, m] = -x
    p = np.zeros((nl, L + 1), np.complex128)
    q = np.zeros((nl, L + 1), np.complex128)
    one_p = np.ones((nl, L + 1), np.complex128)
    one_q = np.ones((nl, L + 1), np.complex128)
    for m in range(L):
        t = -(em1[:, m] + e2l[:, m] * (2.0 - one_p[:, m])) / (em1[:, m] + e2l[:, m] * one_p[:, m])
        alpha = sig[m + 1] / sig[m] if cond else 1.0
        w = alpha * (eta[:, m] / eta[:, m + 1]) * t
        p[:, m + 1] = (1.0 + w) / (1.0 - w)
        one_p[:, m + 1] = 2.0 / (1.0 - w)
    for m in range(L, 0, -1):
        u = -(em1[:, m] + e2l[:, m] * (2.0 - one_q[:, m])) / (em1[:, m] + e2l[:, m] * one_q[:, m])
        beta = sig[m - 1] / sig[m] if cond else 1.0
        w = beta * (eta[:, m] / eta[:, m - 1]) * u
        q[:, m - 1] = (1.0 + w) / (1.0 - w)
        one_q[:, m - 1] = 2.0 / (1.0 - w)
    diag_a = 1.0 / (eta * (em1 + e2l * (1.0 - p * q)))
    return LayerState(np.broadcast_to(sig, (nl, L + 1)), eta, p, q, one_p, one_q, e2l, em1, diag_a)


def _packs(model, breaks, layer, st):
    """build_pack (src/layered.cpp:237-273) for all intervals -> dict of (nlam, nz)."""
    L = model.L
    nz = len(layer)
    nl = st.eta.shape[0]
    P = {k: np.zeros((nl, nz), np.complex128) for k in
         ("eta", "eh", "ehm1", "epa", "epa2m1", "epabm1", "epb2m1", "eqb", "eqabm1", "el2", "elh")}
    h = np.zeros(nz)
    for i in range(nz):
        m = layer[i]
        a, b = breaks[i], breaks[i + 1]
        h[i] = b - a
        eta = st.eta[:, m]
        d, dp, l = model.top_of(m), model.bottom_of(m), model.thickness(m)
        ehm1 = _cexpm1(-eta * h[i])
        P["eta"][:, i] = eta
        P["ehm1"][:, i] = ehm1
        P["eh"][:, i] = 1.0 + ehm1
        P["el2"][:, i] = st.e2l[:, m]
        P["epa"][:, i] = 1.0
        P["eqb"][:, i] = 1.0
        has_p, has_q = m > 0, m < L
        if has_p:
            epam1 = _cexpm1(-eta * (a - d))
            epbm1 = epam1 + ehm1 + epam1 * ehm1
            P["epa"][:, i] = 1.0 + epam1
            P["epa2m1"][:, i] = 2.0 * epam1 + epam1 * epam1
            P["epabm1"][:, i] = epam1 + epbm1 + epam1 * epbm1
            P["epb2m1"][:, i] = 2.0 * epbm1 + epbm1 * epbm1
        if has_q:
            eqbm1 = _cexpm1(-eta * (dp - b))
            eqam1 = eqbm1 + ehm1 + eqbm1 * ehm1
            P["eqb"][:, i] = 1.0 + eqbm1
            P["eqabm1"][:, i] = eqam1 + eqbm1 + eqam1 * eqbm1
        if has_p and has_q:
            P["elh"][:, i] = np.exp(-eta * (2.0 * l - h[i]))
    return P, h


def _factors(layer, st, P, h):
    """make_factors (src/layered.cpp:281-317) for all intervals."""
    lay = np.asarray(layer)
    p, q, A = st.p[:, lay], st.q[:, lay], st.diag_a[:, lay]
    one_p, one_q = st.one_p[:, lay], st.one_q[:, lay]
    eta = P["eta"]
    u = -P["ehm1"]
    Sa = one_p + p * P["epa2m1"]
    Sab = one_p + p * P["epabm1"]
    Mab = (2.0 - one_p) - p * P["epabm1"]
    Dp = one_p + p * P["epb2m1"]
    Tq = one_q + q * P["eqabm1"]
    TMq = (2.0 - one_q) - q * P["eqabm1"]
    F = {}
    F["theta"] = P["eh"] * Sa / Dp
    F["H0"] = u * Sab / (eta * Dp)
    F["H1"] = u * Mab / Dp
    F["J0"] = A * u * Sa * Tq / eta
    F["J1"] = -A * u * Sa * TMq
    Ip = P["epa"] * u / eta
    Iq = P["eqb"] * u / eta
    Sp, Sq = p * Ip * Ip, q * Iq * Iq
    M0 = 2.0 * (h * eta + P["ehm1"]) / (eta * eta)
    P0 = 2.0 * (P["elh"] * u / (eta * eta) - h * P["el2"] / eta)
    F["W00d"] = A * (Sp + Sq + M0 + p * q * P0)
    F["W10d"] = A * eta * (Sq - Sp)
    F["W11d"] = A * (eta * eta * (Sp + Sq) + 2.0 * u - 2.0 * p * q * P["elh"] * u) - 2.0 * h
    F["W20d"] = eta * eta * F["W00d"] - 2.0 * h
    return F


def _fill_table(layer, st, P, F, cond):
    """fill_table (src/layered.cpp:319-378) -> (nlam, 6, nz, nz) in pair order
    (0,0) (1,0) (0,1) (1,1) (2,0) (0,2)."""
    nl, nz = P["eta"].shape
    W = np.zeros((nl, 6, nz, nz), np.complex128)
    for i in range(nz):
        ei2 = P["eta"][:, i] * P["eta"][:, i]
        W[:, 0, i, i] = F["W00d"][:, i]
        W[:, 1, i, i] = F["W10d"][:, i]
        W[:, 2, i, i] = F["W10d"][:, i]
        W[:, 3, i, i] = F["W11d"][:, i]
        W[:, 4, i, i] = F["W20d"][:, i]
        W[:, 5, i, i] = F["W20d"][:, i]
        chain = np.ones(nl, np.complex128)
        for j in range(i + 1, nz):
            base0 = F["H0"][:, i] * chain
            base1 = F["H1"][:, i] * chain
            ej2 = P["eta"][:, j] * P["eta"][:, j]
            b00 = base0 * F["J0"][:, j]
            W[:, 0, i, j] = b00
            W[:, 2, i, j] = base0 * F["J1"][:, j]
            W[:, 5, i, j] = ej2 * b00
            W[:, 1, i, j] = base1 * F["J0"][:, j]
            W[:, 3, i, j] = base1 * F["J1"][:, j]
            W[:, 4, i, j] = ei2 * b00
            chain = chain * F["theta"][:, j]
    for i in range(1, nz):
        for j in range(i):
            ratio = st.sig[:, layer[i]] / st.sig[:, layer[j]] if cond else 1.0
            W[:, 0, i, j] = ratio * W[:, 0, j, i]
            W[:, 1, i, j] = ratio * W[:, 2, j, i]
            W[:, 2, i, j] = ratio * W[:, 1, j, i]
            W[:, 3, i, j] = ratio * W[:, 3, j, i]
            W[:, 4, i, j] = ratio * W[:, 5, j, i]
            W[:, 5, i, j] = ratio * W[:, 4, j, i]
    return W


def moment_tables(model, breaks, omega, lam):
    """vertical_moment_tables (src/layered.cpp:389-395) with the two states of
    MomentMemo::get (src/greens.cpp:116-118) -> (unit, cond), each
    (nlam, 6, nz, nz)."""
    layer = partition_layers(model, breaks)
    su = spectral_state(model, omega, lam, False)
    sc = spectral_state(model, omega, lam, True)
    P, h = _packs(model, breaks, layer, su)
    Fu = _factors(layer, su, P, h)
    Fc = _factors(layer, sc, P, h)
    return _fill_table(layer, su, P, Fu, False), _fill_table(layer, sc, P, Fc, True)


def ntri(nz):
    return nz * (nz + 1) // 2


def tri(k, kp, nz):
    """GreensBlock::tri (include/emie/greens.hpp:61-65)."""
    return k * nz - k * (k - 1) // 2 + (kp - k)


def assemble_block(grid: Grid, omega, oi, oj, den=None, weights=None):
    """assemble_block (src/greens.cpp:150-221) -> dict xx yy zz xy (tri), xz yz (full).

    weights: optional list of six (w, lam) pairs in AB6 order replacing the
    designed filters (lets tests separate the filter design from the
    lambda accumulation)."""
    if abs(oi) >= grid.ny or abs(oj) >= grid.nx:
        raise IndexError("assemble_block: offset outside the grid")
    nz = grid.nz
    geom = pair_geometry(oi, oj, grid.hx, grid.hy)
    R = geom[0]
    if den is None:
        den = filter_denominator()
    ws = weights if weights is not None else [design_weights(geom, a, b, den=den) for a, b in AB6]
    lam = ws[0][1] / R
    tu, tc = moment_tables(grid.model, grid.breaks, omega, lam)
    iwmu = 1j * omega * MU0
    sb = grid.sigma_b[:, None]  # sigma_b[n] of the observation interval
    V1 = iwmu * tu[:, 0]
    V2 = iwmu * tc[:, 0]
    V3 = -tc[:, 3] / sb
    V4 = tc[:, 1] / sb
    V5 = tc[:, 4] / sb  # v_functions (src/layered.cpp:397-408)
    lam3 = lam[:, None, None]
    w00, w20, w02, w11, w10, w01 = (w[0][:, None, None] for w in ws)
    f4 = lam3 * V4
    axz = np.sum(w10 * f4, axis=0)
    ayz = np.sum(w01 * f4, axis=0)
    f2 = (V1 + V3) / lam3
    a00 = np.sum(w00 * (lam3 * V1), axis=0)
    a20 = np.sum(w20 * f2, axis=0)
    a02 = np.sum(w02 * f2, axis=0)
    a11 = np.sum(w11 * f2, axis=0)
    az = np.sum(w00 * (lam3 * (V2 + V5)), axis=0)
    c3, c2, c1 = R ** 3 / (4.0 * PI), R ** 2 / (4.0 * PI), R / (4.0 * PI)
    iu = np.triu_indices(nz)
    blk = {
        "xx": (c3 * a00 + c1 * a20)[iu],
        "yy": (c3 * a00 + c1 * a02)[iu],
        "zz": (c3 * az)[iu],
        "xy": (c1 * a11)[iu],
        "xz": (c2 * axz).reshape(-1),
        "yz": (c2 * ayz).reshape(-1),
    }
    for k, v in blk.items():
        if not np.all(np.isfinite(v)):
            raise FloatingPointError("assemble_block: non-finite " + k)
    return blk


COMPS = ("xx", "yy", "zz", "xy", "xz", "yz")


def block_vector(blk):
    """GreensBlock components concatenated in storage order."""
    return np.concatenate([blk[c] for c in COMPS])


def assemble_operator(grid: Grid, omega):
    """assemble_operator (src/greens.cpp:332-371) -> (ny, nx, 2nz(2nz+1)) offset-major."""
    den = filter_denominator()
    out = np.zeros((grid.ny, grid.nx, 2 * grid.nz * (2 * grid.nz + 1)), np.complex128)
    for oi in range(grid.ny):
        for oj in range(grid.nx):
            out[oi, oj] = block_vector(assemble_block(grid, omega, oi, oj, den))
    return out


# ------------------------------------------------------- toeplitz / apply ---
def smooth_embedding_size(n):
    """src/toeplitz.cpp:18-26."""
    if n < 1:
        raise ValueError("smooth_embedding_size: n < 1")
    c = n
    while True:
        r = c
        for f in (2, 3, 5):
            while r % f == 0:
                r //= f
        if r == 1:
            return c
        c += 1


def _split_block(vec, nz):
    nt, nf = ntri(nz), nz * nz
    o = np.cumsum([0, nt, nt, nt, nt, nf, nf])
    return [vec[..., o[i]:o[i + 1]] for i in range(6)]


def transform_operator(blocks, nx, ny, nz):
    """src/toeplitz.cpp:92-161: blocks (ny, nx, nent) -> (dims, comp[6]) with
    comp[c] of shape (qy*qx, nent_c) (mode-major, toeplitz.hpp:58-61)."""
    if nx <= 0 or ny <= 0 or nz <= 0:
        raise ValueError("transform_operator: empty operator")
    ex, ey = smooth_embedding_size(2 * nx - 1), smooth_embedding_size(2 * ny - 1)
    qx, qy = ex // 2 + 1, ey // 2 + 1
    comps = _split_block(np.asarray(blocks), nz)
    out = []
    for c in range(6):
        sx, sy = PARITY_X[c], PARITY_Y[c]
        v = comps[c]  # (ny, nx, nent_c)
        w = np.zeros((ey, ex, v.shape[-1]), np.complex128)
        w[:ny, :nx] = v
        if nx > 1:
            w[:ny, ex - np.arange(1, nx)] = sx * v[:, 1:]
        if ny > 1:
            w[ey - np.arange(1, ny), :nx] = sy * v[1:, :]
        if nx > 1 and ny > 1:
            w[np.ix_(ey - np.arange(1, ny), ex - np.arange(1, nx))] = sx * sy * v[1:, 1:]
        f = np.fft.fft2(w, axes=(0, 1))
        out.append(f[:qy, :qx].reshape(qy * qx, -1))
    return (ex, ey, qx, qy), out


def _mode_matrix(comp, dims, nz, my, mx):
    """3nz x 3nz coupling of lateral mode (my, mx) as apply rebuilds it
    (toeplitz.cpp:213-250)."""
    ex, ey, qx, qy = dims
    qmy, qmx, fy, fx = my, mx, 1.0, 1.0
    if my > ey // 2:
        qmy, fy = ey - my, -1.0
    if mx > ex // 2:
        qmx, fx = ex - mx, -1.0
    qm = qmy * qx + qmx
    iu = np.triu_indices(nz)

    def sym(t):
        m = np.zeros((nz, nz), np.complex128)
        m[iu] = t
        return m + np.triu(m, 1).T

    xx, yy, zz, xy = (sym(comp[c][qm]) for c in range(4))
    xz = comp[4][qm].reshape(nz, nz)
    yz = comp[5][qm].reshape(nz, nz)
    M = np.zeros((3 * nz, 3 * nz), np.complex128)
    s = slice
    M[s(0, nz), s(0, nz)] = xx
    M[s(0, nz), s(nz, 2 * nz)] = fx * fy * xy
    M[s(0, nz), s(2 * nz, 3 * nz)] = fx * xz
    M[s(nz, 2 * nz), s(0, nz)] = fx * fy * xy
    M[s(nz, 2 * nz), s(nz, 2 * nz)] = yy
    M[s(nz, 2 * nz), s(2 * nz, 3 * nz)] = fy * yz
    M[s(2 * nz, 3 * nz), s(0, nz)] = -fx * xz.T
    M[s(2 * nz, 3 * nz), s(nz, 2 * nz)] = -fy * yz.T
    M[s(2 * nz, 3 * nz), s(2 * nz, 3 * nz)] = zz
    return M


def apply_spectral(comp, dims, nx, ny, nz, v):
    """apply(SpectralOperator) (src/toeplitz.cpp:163-283)."""
    ex, ey, qx, qy = dims
    v = np.asarray(v, np.complex128).reshape(3 * nz, ny, nx)
    pad = np.zeros((3 * nz, ey, ex), np.complex128)
    pad[:, :ny, :nx] = v
    spec = np.fft.fft2(pad, axes=(1, 2))
    out = np.zeros_like(spec)
    for my in range(ey):
        for mx in range(ex):
            out[:, my, mx] = _mode_matrix(comp, dims, nz, my, mx) @ spec[:, my, mx]
    back = np.fft.ifft2(out, axes=(1, 2))  # includes the 1/(ex ey)
    return back[:, :ny, :nx].reshape(-1)


def fetch_block(blocks, nz, oi, oj):
    """src/greens.cpp:295-330 -> (3, 3, nz, nz)."""
    ny, nx = blocks.shape[:2]
    if abs(oi) >= ny or abs(oj) >= nx:
        raise IndexError("fetch_block: offset out of range")
    b = _split_block(blocks[abs(oi), abs(oj)], nz)
    sx = -1.0 if oj < 0 else 1.0
    sy = -1.0 if oi < 0 else 1.0
    iu = np.triu_indices(nz)

    def sym(t):
        m = np.zeros((nz, nz), np.complex128)
        m[iu] = t
        return m + np.triu(m, 1).T

    F = np.zeros((3, 3, nz, nz), np.complex128)
    F[0, 0], F[1, 1], F[2, 2] = sym(b[0]), sym(b[1]), sym(b[2])
    F[0, 1] = F[1, 0] = sx * sy * sym(b[3])
    F[0, 2] = sx * b[4].reshape(nz, nz)
    F[1, 2] = sy * b[5].reshape(nz, nz)
    F[2, 0] = -F[0, 2].T
    F[2, 1] = -F[1, 2].T
    return F


def dense_apply(blocks, nx, ny, nz, v):
    """dense_reference_apply (src/toeplitz.cpp:285-312)."""
    if nx * ny * nz > 4096:
        raise ValueError("dense_reference_apply: grid too large")
    v = np.asarray(v, np.complex128).reshape(3, nz, ny, nx)
    out = np.zeros_like(v)
    for oi in range(-(ny - 1), ny):
        for oj in range(-(nx - 1), nx):
            F = fetch_block(blocks, nz, oi, oj)
            for iy in range(max(0, oi), min(ny, ny + oi)):
                for ix in range(max(0, oj), min(nx, nx + oj)):
                    src = v[:, :, iy - oi, ix - oj]  # (3, nz)
                    out[:, :, iy, ix] += np.einsum("abkl,bl->ak", F, src)
    return out.reshape(-1)


def system_diagonals(grid: Grid):
    """build_system (src/cie.cpp:24-54) with contrast_coefficients (9-22)."""
    nz = grid.nz
    s = np.zeros((nz, grid.ny, grid.nx), np.complex128)
    r1 = np.zeros((nz, grid.ny, grid.nx))
    r2 = np.zeros_like(s)
    for iz in range(nz):
        sb = grid.sigma_b[iz]
        if not sb.real > 0.0:
            raise ValueError("build_system: interval without conduction")
        sq = math.sqrt(sb.real)
        sa = grid.sigma_a[iz]
        g = (sa - sb) / (sa + np.conj(sb))
        if np.any(~(np.abs(g) < 1.0)):
            raise ArithmeticError("contrast coefficients: contraction factor reaches one")
        s[iz] = 1.0 - g
        r1[iz] = 2.0 / grid.volume(iz) * sq
        r2[iz] = -sq * g
    return s.reshape(-1), r1.reshape(-1), r2.reshape(-1)


def apply_system(diag, applyB, u):
    """apply(SystemOperator) (src/cie.cpp:56-73); applyB maps a field to B v."""
    s, r1, r2 = diag
    u = np.asarray(u, np.complex128).reshape(3, -1)
    out = np.asarray(applyB((r2[None, :] * u).reshape(-1))).reshape(3, -1)
    return (s[None, :] * u + r1[None, :] * out).reshape(-1)


def _make_rotation(f, g):
    """src/cie.cpp:100-113."""
    if g == 0:
        return 1.0, 0j
    if f == 0:
        return 0.0, np.conj(g) / abs(g)
    t = math.sqrt(abs(f) ** 2 + abs(g) ** 2)
    return abs(f) / t, f / abs(f) * np.conj(g) / t


def fgmres(apply_a, rhs, tol=1e-8, restart=40, max_iters=500):
    """Flexible restarted GMRES, MGS twice (src/cie.cpp:117-238), no
    preconditioner. -> (x, report dict)."""
    if not tol > 0 or restart < 1 or max_iters < 1:
        raise ValueError("fgmres: bad solver configuration")
    rhs = np.asarray(rhs, np.complex128).reshape(-1)
    x = np.zeros_like(rhs)
    rep = {"status": "max_iterations", "iterations": 0, "residual": 0.0, "history": []}
    bnorm = np.linalg.norm(rhs)
    if bnorm == 0.0:
        rep["status"] = "converged"
        return x, rep
    m = restart
    r = rhs.copy()
    rnorm = bnorm
    it = 0
    broke = False
    while it < max_iters:
        V = [r / rnorm]
        H = np.zeros((m, m + 1), np.complex128)  # H[j] = column j
        cs = np.zeros(m)
        sn = np.zeros(m, np.complex128)
        g = np.zeros(m + 1, np.complex128)
        g[0] = rnorm
        cols = 0
        for j in range(m):
            if not it < max_iters:
                break
            it += 1
            w = apply_a(V[j])
            wn0 = np.linalg.norm(w)
            hj = H[j]
            for _ in range(2):
                for i in range(j + 1):
                    hc = np.vdot(V[i], w)
                    w = w - hc * V[i]
                    hj[i] += hc
            hnext = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * hj[i] + sn[i] * hj[i + 1]
                hj[i + 1] = -np.conj(sn[i]) * hj[i] + cs[i] * hj[i + 1]
                hj[i] = t
            if hnext <= 1e-13 * max(wn0, 1e-300):
                colmax = max([hnext] + [abs(hj[i]) for i in range(j + 1)])
                if abs(hj[j]) > 1e-13 * max(colmax, 1e-300):
                    cols = j + 1
                else:
                    cols = j
                    broke = True
                    rep["history"].append(rnorm / bnorm)
                break
            hj[j + 1] = hnext
            V.append(w / hnext)
            cs[j], sn[j] = _make_rotation(hj[j], hnext)
            t = cs[j] * hj[j] + sn[j] * hj[j + 1]
            hj[j + 1] = 0
            hj[j] = t
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            cols = j + 1
            est = abs(g[j + 1]) / bnorm
            rep["history"].append(est)
            if est <= tol:
                break
        if cols > 0:
            y = np.zeros(cols, np.complex128)
            for k in range(cols - 1, -1, -1):
                acc = g[k]
                for l in range(k + 1, cols):
                    acc -= H[l, k] * y[l]
                y[k] = acc / H[k, k]
            for k in range(cols):
                x = x + y[k] * V[k]
        r = rhs - apply_a(x)
        rnorm = np.linalg.norm(r)
        if rnorm / bnorm <= tol:
            rep["status"] = "converged"
            break
        if broke:
            rep["status"] = "breakdown"
            break
    if broke and rnorm / bnorm <= tol:
        rep["status"] = "converged"
    rep["iterations"] = it
    rep["residual"] = rnorm / bnorm
    return x, rep
