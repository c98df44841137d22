"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs here (CPU container) against oracle/_ref/libemie_ref_capi.so, which
oracle/Makefile compiles from the reference's own sources under
/root/reference. The fixtures travel with the repo; the GPU box never needs
/root/reference.

    python tests/golden/make_golden.py

Fixtures
  toeplitz_{single,tiny,small,large}.npz  the grids of the reference's own
      test_toeplitz.cpp:25-61 (contrast model, 200 m x 260 m cells, T = 50 s):
      compressed blocks, spectra, seeded fields and the reference's
      apply(SpectralOperator), dense_reference_apply, build_system
      diagonals and apply(SystemOperator) on a seeded anomaly.
  cfg1.npz  BASELINE config 1 (16x16x8): blocks, spectra, applies, and
      solve_cie for the x/y plane-wave right-hand sides at tol 1e-6 / 1e-10.
  filters.npz  FilterDesigner weights for several geometries.
  tables.npz   vertical moment tables at several lambda (three_layer model of
      test_layered.cpp:22-27).
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import ref_binding as R  # noqa: E402
from paper_1512_06126_b200 import configs, normal_field  # noqa: E402

CONTRAST = ([0.0, 400.0], [0.0, 0.01, 0.1])  # test_toeplitz.cpp:25-30
TOEPLITZ = {
    "single": (1, 1, [0.0, 200.0, 400.0, 700.0]),  # test_toeplitz.cpp:188-193
    "tiny": (2, 2, [0.0, 200.0, 400.0]),            # :47-50
    "small": (4, 4, [0.0, 200.0, 400.0, 700.0]),    # :52-55
    "large": (6, 5, [0.0, 150.0, 300.0, 400.0, 700.0]),  # :57-61
}


def rand_field(rng, n):
    return rng.uniform(-1.0, 1.0, n) + 1j * rng.uniform(-1.0, 1.0, n)


def toeplitz_fixture(name, nx, ny, breaks):
    tops, sig = CONTRAST
    omega = 2.0 * np.pi / 50.0
    nz = len(breaks) - 1
    rng = np.random.default_rng({"single": 11, "tiny": 12, "small": 1234, "large": 1235}[name])
    # seeded anomaly for the system operator: log-uniform around the host layer
    sb = np.array([0.01 if b < 400.0 else 0.1 for b in breaks[:-1]])
    sa = (sb[:, None, None] * 10.0 ** rng.uniform(-2.0, 2.0, (nz, ny, nx))).astype(np.complex128)
    case = R.RefCase(tops, sig, breaks, nx, ny, 200.0, 260.0, omega, sa)
    blocks, spec, dims = case.build()
    n = 3 * nx * ny * nz
    vecs = np.stack([rand_field(rng, n) for _ in range(3)])
    applyB = np.stack([case.apply("spectral", v) for v in vecs])
    dense = np.stack([case.apply("dense", v) for v in vecs])
    applyA = np.stack([case.apply("system", v) for v in vecs])
    s, r1, r2 = case.diagonals()
    np.savez_compressed(HERE / f"toeplitz_{name}.npz", tops=tops, sigma=np.array(sig, np.complex128),
                        breaks=breaks, nx=nx, ny=ny, hx=200.0, hy=260.0, omega=omega,
                        sigma_a=sa, blocks=blocks, spec=spec, dims=np.array(dims), vecs=vecs,
                        applyB=applyB, denseB=dense, applyA=applyA, s=s, r1=r1, r2=r2)
    print(f"toeplitz_{name}: dims {dims}")


def cfg1_fixture():
    c = configs.config(1)
    case = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a)
    t0 = time.time()
    blocks, spec, dims = case.build()
    tb = time.time() - t0
    rng = np.random.default_rng(77)
    n = 3 * c.cells()
    vecs = np.stack([rand_field(rng, n) for _ in range(2)])
    applyB = np.stack([case.apply("spectral", v) for v in vecs])
    applyA = np.stack([case.apply("system", v) for v in vecs])
    rhs = np.stack([normal_field.build_rhs(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.omega, p)
                    for p in "xy"])
    sol = {}
    for tol in (1e-6, 1e-10):
        xs, reps = [], []
        for b in rhs:
            x, rep = case.solve(b, tol)
            xs.append(x)
            reps.append(rep)
        sol[tol] = (np.stack(xs), reps)
    np.savez_compressed(HERE / "cfg1.npz", tops=c.tops, sigma=np.array(c.sigma, np.complex128),
                        breaks=c.breaks, nx=c.nx, ny=c.ny, hx=c.hx, hy=c.hy, omega=c.omega,
                        sigma_a=c.sigma_a, blocks=blocks, spec=spec, dims=np.array(dims),
                        vecs=vecs, applyB=applyB, applyA=applyA, rhs=rhs,
                        x_tol6=sol[1e-6][0], x_tol10=sol[1e-10][0],
                        iters_tol6=np.array([r["iterations"] for r in sol[1e-6][1]]),
                        iters_tol10=np.array([r["iterations"] for r in sol[1e-10][1]]),
                        resid_tol6=np.array([r["residual"] for r in sol[1e-6][1]]),
                        hist_tol6_x=np.array(sol[1e-6][1][0]["history"]),
                        greens_seconds=tb)
    print(f"cfg1: dims {dims}, build {tb:.2f}s, iters {[r['iterations'] for r in sol[1e-6][1]]}")


def filters_fixture():
    geoms = [(0, 0, 1.0, 1.0), (0, 1, 200.0, 200.0), (1, 2, 200.0, 260.0), (-1, 2, 1.3, 0.7),
             (0, 5, 100.0, 100.0), (7, 3, 250.0, 250.0), (15, 15, 500.0, 500.0)]
    ab = [(0, 0), (2, 0), (0, 2), (1, 1), (1, 0), (0, 1)]
    W = np.zeros((len(geoms), 6, 451))
    lam = None
    for i, (oi, oj, hx, hy) in enumerate(geoms):
        for k, (a, b) in enumerate(ab):
            W[i, k], lam = R.design_weights(oi, oj, hx, hy, a, b)
    np.savez_compressed(HERE / "filters.npz", geoms=np.array(geoms), W=W, lam=lam)
    print("filters: ok")


def tables_fixture():
    tops, sig = [0.0, 50.0, 150.0], [0.0, 0.02, 0.5, 0.05]  # test_layered.cpp:22-27
    breaks = [0.0, 25.0, 50.0, 90.0, 150.0, 220.0]
    omega = 2.0 * np.pi / 10.0
    lams = [1e-5, 1e-3, 0.02, 0.3, 5.0]
    T = np.stack([R.moment_tables(tops, sig, breaks, omega, l) for l in lams])
    np.savez_compressed(HERE / "tables.npz", tops=tops, sigma=np.array(sig, np.complex128),
                        breaks=breaks, omega=omega, lams=lams, T=T)
    print("tables: ok")


if __name__ == "__main__":
    R.build()
    for name, (nx, ny, br) in TOEPLITZ.items():
        toeplitz_fixture(name, nx, ny, br)
    filters_fixture()
    tables_fixture()
    cfg1_fixture()
