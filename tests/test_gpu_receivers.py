"""Receiver-side integrals and fields (SPEC.md receiver_green_integrals /
reconstruct_fields; the reference has only placeholders, src/receiver.cpp:1,
so parity rests on the SPEC's own checks and on the device Green's blocks):

* homogeneous whole space: int_cell G^E and int_cell G^H against brute
  Gauss cubature of the analytic whole-space dyadic (1 + grad grad / k^2)
  i w mu0 e^{-kappa r} / (4 pi r) and its curl, <= 1e-5 (SPEC's bar), for
  receivers above, below, beside the cells at their depths and on their
  face planes;
* layered medium: the receiver tensor averaged over an observation cell
  reproduces the Galerkin block B_n^m of the device Green's build for that
  pair of cells (paper Eq. slae_matricies: B = int_n int_m G^E), at the
  filter accuracy of the two independent lateral quadratures;
* fields: zero contrast gives zero anomalous field; linearity in U."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1512_06126_b200 as emie

pytestmark = pytest.mark.gpu
MU0 = 1.2566370614359172e-06


def _gl(n, a, b):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (b - a) * x + 0.5 * (a + b), 0.5 * (b - a) * w


def wholespace_tensors(rec, box, sigma, omega, n=24, split=2):
    """Brute cubature over the box [(x0,x1),(y0,y1),(z0,z1)] of the whole-space
    G^E and G^H (receiver-coordinate derivatives), split^3 sub-boxes x n^3 points."""
    kap = np.sqrt(-1j * omega * MU0 * sigma)
    kap = kap if kap.real > 0 else -kap
    k2 = 1j * omega * MU0 * sigma
    GE = np.zeros((3, 3), complex)
    GH = np.zeros((3, 3), complex)
    edges = [np.linspace(a, b, split + 1) for a, b in box]
    for i in range(split):
        for j in range(split):
            for l in range(split):
                X, WX = _gl(n, edges[0][i], edges[0][i + 1])
                Y, WY = _gl(n, edges[1][j], edges[1][j + 1])
                Z, WZ = _gl(n, edges[2][l], edges[2][l + 1])
                x, y, z = np.meshgrid(X, Y, Z, indexing="ij")
                w = (WX[:, None, None] * WY[None, :, None] * WZ[None, None, :])
                d = np.stack([rec[0] - x, rec[1] - y, rec[2] - z])
                r = np.sqrt(np.sum(d * d, axis=0))
                phi = np.exp(-kap * r) / r
                d1 = -(kap + 1.0 / r) * phi
                d2 = (kap * kap + 2 * kap / r + 2 / (r * r)) * phi
                for a in range(3):
                    for bb in range(3):
                        dd = d2 * d[a] * d[bb] / r ** 2 + d1 * ((a == bb) / r - d[a] * d[bb] / r ** 3)
                        GE[a, bb] += np.sum(w * (1j * omega * MU0 / (4 * np.pi)) * ((a == bb) * phi + dd / k2))
                grad = [d1 * d[q] / r for q in range(3)]
                eps = {(0, 1, 2): 1, (1, 2, 0): 1, (2, 0, 1): 1, (0, 2, 1): -1, (2, 1, 0): -1, (1, 0, 2): -1}
                for (a, kq, bb), sgn in eps.items():
                    GH[a, bb] += sgn * np.sum(w * grad[kq]) / (4 * np.pi)
    return GE, GH


@pytest.mark.parametrize("rec", [(-350.0, 80.0, -30.0), (520.0, -260.0, 0.0), (50.0, 40.0, -220.0),
                                 (800.0, 700.0, 450.0), (520.0, -260.0, 50.0), (520.0, -260.0, 100.0),
                                 (520.0, -260.0, 400.0), (-20.0, 300.0, 175.0)])
def test_wholespace_receiver_integrals(torch_cuda, rec):
    sigma, omega = 0.02, 2 * np.pi * 3.0
    model = emie.LayeredModel([0.0], [sigma, sigma])  # the same conductivity above and below: a whole space
    breaks = [0.0, 100.0, 250.0, 400.0]
    grid = emie.make_grid(model, breaks, 3, 2, 150.0, 120.0, x0=-100.0, y0=-60.0)
    got = emie.receiver_tensors(grid, model, omega, rec, 1, 1)
    box_xy = ((-100.0 + 150.0, -100.0 + 300.0), (-60.0 + 120.0, -60.0 + 240.0))
    for k in range(3):
        GE, GH = wholespace_tensors(rec, (*box_xy, (breaks[k], breaks[k + 1])), sigma, omega)
        se, sh = np.max(np.abs(GE)), np.max(np.abs(GH))
        ee = np.max(np.abs(got[k, 0] - GE)) / se
        eh = np.max(np.abs(got[k, 1] - GH)) / sh
        assert ee <= 1e-5 and eh <= 1e-5, (rec, k, ee, eh)


def test_receiver_tensor_averages_to_galerkin_block(torch_cuda):
    """B_n^m (device Green's build) = int over cell n of the receiver tensor of
    cell m: 4 x 4 x 4 Gauss points in an observation cell two cells away."""
    model = emie.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])
    breaks = [0.0, 150.0, 300.0, 400.0, 700.0]
    hx, hy = 200.0, 260.0
    omega = 2 * np.pi / 10.0
    big = emie.make_grid(model, breaks, 6, 6, hx, hy)
    oi, oj = 2, 3
    blk = emie.assemble_block(big, model, omega, oi, oj)[0]
    nz = 4
    nt = nz * (nz + 1) // 2
    # the source column alone (receivers outside it), observation cell at (oj hx, oi hy)
    src = emie.make_grid(model, breaks, 1, 1, hx, hy)
    X, WX = _gl(4, oj * hx, (oj + 1) * hx)
    Y, WY = _gl(4, oi * hy, (oi + 1) * hy)
    for k in range(nz):
        Z, WZ = _gl(4, breaks[k], breaks[k + 1])
        acc = np.zeros((nz, 3, 3), complex)
        for x, wx in zip(X, WX):
            for y, wy in zip(Y, WY):
                for z, wz in zip(Z, WZ):
                    acc += wx * wy * wz * emie.receiver_tensors(src, model, omega, (x, y, z), 0, 0)[:, 0]
        scale = np.max(np.abs(blk))
        for kp in range(nz):
            lo, hi = min(k, kp), max(k, kp)
            t = lo * nz - lo * (lo - 1) // 2 + (hi - lo)
            want = {(0, 0): blk[t], (1, 1): blk[nt + t], (2, 2): blk[2 * nt + t], (0, 1): blk[3 * nt + t],
                    (0, 2): blk[4 * nt + k * nz + kp], (1, 2): blk[4 * nt + nz * nz + k * nz + kp]}
            for (a, b), w in want.items():
                assert abs(acc[kp, a, b] - w) <= 2e-5 * scale, (k, kp, a, b, acc[kp, a, b], w)
            # the z-row couplings: zx(k, kp) = -xz(kp, k) of the stored block
            assert abs(acc[kp, 2, 0] + blk[4 * nt + kp * nz + k]) <= 2e-5 * scale


def test_receiver_fields_zero_contrast_and_linearity(torch_cuda):
    model = emie.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])
    grid = emie.make_grid(model, [100.0, 200.0, 300.0], 4, 3, 200.0, 200.0)
    omega = 2 * np.pi / 10.0
    rng = np.random.default_rng(3)
    n = 3 * grid.nx * grid.ny * grid.nz
    U = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
    recs = np.array([[-150.0, 100.0, 0.0], [400.0, 300.0, 50.0], [900.0, -40.0, 0.0]])
    f0 = emie.receiver_fields(grid, model, omega, U, recs)
    assert np.all(f0 == 0)  # sigma_a = sigma_b everywhere: no scattering currents
    grid.sigma_a[1, 1:3, 1:3] = 0.5
    f = emie.receiver_fields(grid, model, omega, U, recs)
    f1 = emie.receiver_fields(grid, model, omega, U[:1], recs)
    f2 = emie.receiver_fields(grid, model, omega, 2.0 * U[1:], recs)
    assert np.allclose(f[:, 0], f1[:, 0], rtol=1e-13, atol=0)
    assert np.allclose(2.0 * f[:, 1], f2[:, 0], rtol=1e-13, atol=1e-30)
    with pytest.raises(emie.InvalidArgument):
        emie.receiver_fields(grid, model, omega, U, [[100.0, 100.0, 150.0]])  # inside the anomaly
