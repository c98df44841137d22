"""Plane-wave normal field and CIE right-hand side.

The reference leaves this stage as a placeholder (src/normal_field.cpp:1),
so there is no reference arithmetic to match; one shared host routine feeds
both the oracle and the B200 solver. It is a 1-D,
O(layers) computation per frequency and stays on the host.

Convention: fields ~ e^{-i omega t} with eta_m = sqrt(-i omega mu0 sigma_m),
Re eta > 0 (the lambda = 0 limit of build_spectral_state, layered.cpp:87-89);
unit tangential electric field at z = 0; the lower halfspace carries only
the decaying mode. Inside layer m (top zt, bottom zb, thickness l):
    E(z) = D [ e^{-eta (z - zt)} + rho e^{-eta l} e^{-eta (zb - z)} ]
with rho = (eta + Y_b) / (eta - Y_b) fixed by the admittance Y = E'/E at the
bottom; every exponential has a non-positive real exponent.
"""
from __future__ import annotations

import cmath

import numpy as np

MU0 = 1.2566370614359172e-06


def _cexpm1(x: complex) -> complex:
    """e^x - 1 without cancellation (the form of layered.cpp:19-25)."""
    import math
    em = math.expm1(x.real)
    s = math.sin(0.5 * x.imag)
    return complex(em * math.cos(x.imag) - 2.0 * s * s, (em + 1.0) * math.sin(x.imag))


def _layers(tops, sigma, omega):
    L = len(tops)
    eta = []
    for m in range(L + 1):
        s = complex(sigma[m])
        if s.real < 1e-9:
            s = complex(1e-9, s.imag)
        e = cmath.sqrt(-1j * omega * MU0 * s)
        eta.append(-e if e.real < 0 else e)
    return eta


def profile(tops, sigma, omega):
    """-> list of per-layer (zt, l, D, rho, eta) for layers 1..L (l = inf for
    the lower halfspace), normalised to E(0) = 1 with z = 0 the top of layer 1."""
    L = len(tops)
    eta = _layers(tops, sigma, omega)
    # admittance from the bottom up
    Y = [None] * (L + 1)
    rho = [0j] * (L + 1)
    Yb = -eta[L]
    Y[L] = Yb
    for m in range(L - 1, 0, -1):
        l = tops[m] - tops[m - 1]
        e = eta[m]
        r = (e + Yb) / (e - Yb)
        rho[m] = r
        q = r * cmath.exp(-2.0 * e * l)
        Yb = e * (-1.0 + q) / (1.0 + q)
        Y[m] = Yb
    out = []
    Et = 1.0 + 0j  # E at the surface (top of layer 1)
    for m in range(1, L + 1):
        e = eta[m]
        zt = tops[m - 1]
        if m == L:
            out.append((zt, np.inf, Et, 0j, e, eta[0]))
            break
        l = tops[m] - tops[m - 1]
        el = cmath.exp(-e * l)
        D = Et / (1.0 + rho[m] * el * el)
        out.append((zt, l, D, rho[m], e, eta[0]))
        Et = D * el * (1.0 + rho[m])
    return out


def _air(prof, z, deriv, tops=None):
    """Above the surface (z < 0): the upper halfspace continues E and E' of
    z = 0 (both modes; sigma_air floored to 1e-9, so nearly linear in z)."""
    e0, d0 = field_at(prof, 0.0), derivative_at(prof, 0.0)
    ea = prof[0][5] if len(prof[0]) > 5 else None
    if ea is None or ea == 0:
        return d0 if deriv else e0 + d0 * z
    c, s = cmath.cosh(ea * z), cmath.sinh(ea * z)
    if deriv:
        return e0 * ea * s + d0 * c
    return e0 * c + d0 / ea * s


def field_at(prof, z):
    if z < 0.0:
        return _air(prof, z, False)
    for zt, l, D, r, e, *_ in prof:
        if z >= zt and (z < zt + l or np.isinf(l)):
            if np.isinf(l):
                return D * cmath.exp(-e * (z - zt))
            return D * (cmath.exp(-e * (z - zt)) + r * cmath.exp(-e * l) * cmath.exp(-e * (zt + l - z)))
    raise ValueError("depth above the surface")


def derivative_at(prof, z):
    """dE/dz of the profile at depth z (on an interface, the layer below; z < 0:
    the upper halfspace)."""
    if z < 0.0:
        return _air(prof, z, True)
    for zt, l, D, r, e, *_ in prof:
        if z >= zt and (z < zt + l or np.isinf(l)):
            if np.isinf(l):
                return -e * D * cmath.exp(-e * (z - zt))
            return e * D * (-cmath.exp(-e * (z - zt)) + r * cmath.exp(-e * l) * cmath.exp(-e * (zt + l - z)))
    raise ValueError("depth above the surface")


def magnetic_at(prof, z, omega):
    """Tangential H^N of the profile (Faraday, fields ~ e^{-i omega t}):
    H_y = (dE_x/dz) / (i omega mu0) for an x-polarised E (and H_x = -(dE_y/dz) /
    (i omega mu0) for a y-polarised one)."""
    return derivative_at(prof, z) / (1j * omega * MU0)


def normal_fields(tops, sigma, omega, points):
    """Total normal fields at points (n, 3) for the two plane-wave
    polarisations -> E, H each (n, 2, 3) complex: pol x has E = (E(z), 0, 0),
    H = (0, E'/(i w mu0), 0); pol y has E = (0, E(z), 0), H = (-E'/(i w mu0), 0, 0)."""
    prof = profile(tops, sigma, omega)
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    E = np.zeros((len(pts), 2, 3), np.complex128)
    H = np.zeros_like(E)
    for i, (_, _, z) in enumerate(pts):
        e, h = field_at(prof, z), magnetic_at(prof, z, omega)
        E[i, 0, 0], H[i, 0, 1] = e, h
        E[i, 1, 1], H[i, 1, 0] = e, -h
    return E, H


def surface_impedance(tops, sigma, omega):
    """Z = E_x / H_y at z = 0+ (earth side, SPEC.md DESIGN DECISIONS) of the
    1-D background -> (Z, rho_a = |Z|^2 / (omega mu0), phase in degrees). The
    phase is reported in the e^{+i omega t} MT convention, arg(conj Z), so a
    uniform halfspace gives +45 degrees (SPEC.md normal_field_profile)."""
    prof = profile(tops, sigma, omega)
    z = 1.0 / magnetic_at(prof, 0.0, omega)  # E(0) = 1
    return z, abs(z) ** 2 / (omega * MU0), float(np.degrees(np.angle(np.conj(z))))


def interval_average(prof, a, b):
    """(1/(b-a)) * integral of E over [a, b] inside one layer."""
    h = b - a
    for zt, l, D, r, e, *_ in prof:
        if a >= zt - 1e-9 and (np.isinf(l) or b <= zt + l + 1e-7 * (1.0 + abs(b))):
            g = -_cexpm1(-e * h) / e  # (1 - e^{-eta h}) / eta
            down = cmath.exp(-e * (a - zt)) * g
            if np.isinf(l):
                return D * down / h
            up = r * cmath.exp(-e * l) * cmath.exp(-e * (zt + l - b)) * g
            return D * (down + up) / h
    raise ValueError("interval straddles a layer")


def build_rhs(tops, sigma, breaks, nx, ny, omega, polarization: str):
    """U0_n = sqrt(Re sigma_b^n) * cell average of E^N for
    an x- or y-polarised plane wave -> GridVector-layout complex array."""
    prof = profile(tops, sigma, omega)
    nz = len(breaks) - 1
    u = np.zeros((3, nz, ny, nx), np.complex128)
    c = {"x": 0, "y": 1}[polarization]
    import bisect
    for iz in range(nz):
        m = bisect.bisect_right(list(tops), breaks[iz])
        sb = complex(sigma[m])
        sb = max(sb.real, 1e-9)
        u[c, iz] = np.sqrt(sb) * interval_average(prof, breaks[iz], breaks[iz + 1])
    return u.reshape(-1)
