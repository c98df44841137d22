"""Plane-wave normal field and CIE right-hand side (the
reference has only a placeholder, src/normal_field.cpp:1, so these are the
SPEC's own examples and properties, with an independently written 1-D
impedance recursion as the oracle for the layered case)."""
import cmath
import math

import numpy as np
import pytest

from paper_1512_06126_b200 import normal_field as NF

MU0 = NF.MU0


def wait_recursion(thick, sigma, omega):
    """Surface impedance of a layered earth by the classical bottom-up
    recursion Z_m = z_m (Z_{m+1} + z_m t_m) / (z_m + Z_{m+1} t_m),
    z_m = -i omega mu0 / k_m, k_m = sqrt(-i omega mu0 sigma_m), t_m =
    tanh(k_m h_m) (fields ~ e^{-i omega t}). thick: earth layers above the
    basement; sigma: their conductivities + the basement's."""
    k = [cmath.sqrt(-1j * omega * MU0 * s) for s in sigma]
    k = [-x if x.real < 0 else x for x in k]
    zi = [-1j * omega * MU0 / x for x in k]
    Z = zi[-1]
    for m in range(len(thick) - 1, -1, -1):
        t = cmath.tanh(k[m] * thick[m])
        Z = zi[m] * (Z + zi[m] * t) / (zi[m] + Z * t)
    return Z  # E_x / H_y with H_y = E_x' / (i omega mu0)


@pytest.mark.parametrize("sigma,period", [(0.01, 1.0), (1.0, 100.0), (3e-4, 0.01)])
def test_halfspace_apparent_resistivity_and_phase(sigma, period):
    omega = 2 * math.pi / period
    z, rho, phi = NF.surface_impedance([0.0], [0.0, sigma], omega)
    assert abs(rho * sigma - 1.0) <= 1e-3
    assert abs(phi - 45.0) <= 0.05


def test_commemi_background_matches_independent_recursion():
    # SPEC.md normal_field_profile: 1e-3 and 1e-4 S/m layers of 1 and 6.5 km over 0.1 S/m, T = 1 s
    tops, sig = [0.0, 1000.0, 7500.0], [0.0, 1e-3, 1e-4, 0.1]
    for period in (0.1, 1.0, 100.0):
        omega = 2 * math.pi / period
        z, rho, phi = NF.surface_impedance(tops, sig, omega)
        want = wait_recursion([1000.0, 6500.0], sig[1:], omega)
        assert abs(z - want) <= 1e-10 * abs(want)
        assert rho > 0 and -180.0 < phi <= 180.0


def test_continuity_across_interfaces():
    tops, sig = [0.0, 500.0, 2500.0, 7500.0], [0.0, 1e-3, 0.05, 3e-3, 1.0]
    omega = 2 * math.pi * 0.3
    prof = NF.profile(tops, sig, omega)
    assert abs(NF.field_at(prof, 0.0) - 1.0) <= 1e-14
    for zi in tops[1:]:
        above, below = zi * (1 - 1e-15), zi
        for f in (NF.field_at, NF.derivative_at):
            a, b = f(prof, above), f(prof, below)
            # E and E' continuous (the layers' conductivities differ: E' is the H field)
            assert abs(a - b) <= 1e-10 * max(abs(a), abs(b)), (f.__name__, zi, a, b)
    # decay in the basement: only the decaying mode
    d1, d2 = NF.field_at(prof, 8000.0), NF.field_at(prof, 9000.0)
    assert abs(d2) < abs(d1)


def test_rhs_components_and_sqrt_sigma_scaling():
    tops, sig = [0.0, 1000.0, 11000.0], [0.0, 0.01, 0.001, 0.1]
    breaks = list(np.arange(0.0, 2000.0 + 1, 250.0))
    omega = 2 * math.pi * 0.1
    nx, ny, nz = 3, 2, len(breaks) - 1
    ux = NF.build_rhs(tops, sig, breaks, nx, ny, omega, "x").reshape(3, nz, ny, nx)
    uy = NF.build_rhs(tops, sig, breaks, nx, ny, omega, "y").reshape(3, nz, ny, nx)
    assert np.all(ux[1:] == 0) and np.all(uy[0] == 0) and np.all(uy[2] == 0)
    assert np.array_equal(ux[0], uy[1])  # the 1-D profile does not know the polarisation
    prof = NF.profile(tops, sig, omega)
    for iz in range(nz):
        sb = 0.01 if breaks[iz] < 1000.0 else 0.001
        avg = NF.interval_average(prof, breaks[iz], breaks[iz + 1])
        # U0 = sqrt(Re sigma_b) * cell average: doubling Re sigma_b scales it by sqrt(2)
        assert np.allclose(ux[0, iz], math.sqrt(sb) * avg, rtol=1e-15, atol=0)
        assert np.all(ux[0, iz] == ux[0, iz, 0, 0])  # laterally uniform
    # the cell average against a fine midpoint rule of E over the interval
    a, b = breaks[1], breaks[2]
    zs = a + (np.arange(20000) + 0.5) * (b - a) / 20000
    brute = np.mean([NF.field_at(prof, z) for z in zs])
    assert abs(NF.interval_average(prof, a, b) - brute) <= 1e-8 * abs(brute)
