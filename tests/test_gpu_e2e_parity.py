"""End-to-end parity at the benchmark shapes:

* config 3 (the bench workload): apply(SystemOperator) and
  apply(SpectralOperator) on the DEVICE-BUILT operator -- the 256-point TMA
  lateral passes and the octant FP64 tensor-core contraction the bench times
  -- against the reference's own applies (src/cie.cpp:56-73,
  src/toeplitz.cpp:163-283) on the same compressed blocks, at 1e-12 of max
  (test_toeplitz.cpp:314-325's bar);
* config 2, the full chain: device Green's build + both plane-wave
  polarisations solved on the device at tol 1e-6, against the reference's
  own build + solve_cie (cie.cpp:240-249). The fields must lie within the
  reference's own arithmetic envelope (its FMA-contracted build's distance
  from it, oracle/ref_envelope.py), the iteration counts within +-2 of its;
* config 2, the solver alone: the device FGMRES on the reference's operator
  against the reference's solve_cie: 1e-8 (CGS2 vs the reference's MGS2:
  the same Krylov space in exact arithmetic)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1512_06126_b200 as emie
import ref_binding as R
import ref_envelope as RE
from paper_1512_06126_b200 import configs, normal_field as NF

pytestmark = pytest.mark.gpu


def _setup(k):
    c = configs.config(k)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
    grid.sigma_a[...] = c.sigma_a
    return c, model, grid


def test_cfg3_applies_on_device_built_operator(torch_cuda):
    c, model, grid = _setup(3)
    op = emie.assemble_operator(grid, model, c.omega, keep_blocks=True)
    assert emie.xy_symmetric(op), "the bench's octant contraction is not selected"
    blocks = op.blocks().reshape(c.ny, c.nx, -1)
    ref = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a)
    ref.set_operator(blocks)
    sysop = emie.build_system(grid, op)
    rng = np.random.default_rng(1234)
    n = 3 * c.cells()
    for _ in range(2):
        u = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        for which, dev_op in (("system", sysop), ("spectral", op)):
            want = ref.apply(which, u)
            got = emie.apply(dev_op, u)
            err = np.max(np.abs(got - want)) / np.max(np.abs(want))
            assert err <= 1e-12, f"cfg3 apply({which}) vs reference: {err:.2e}"


def _rhs(c):
    return np.stack([NF.build_rhs(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.omega, p).reshape(-1) for p in "xy"])


def test_cfg2_chain_within_reference_envelope(torch_cuda):
    c, model, grid = _setup(2)
    rhs = _rhs(c)
    op = emie.assemble_operator(grid, model, c.omega)
    x, reps = emie.solve_cie(grid, model, op, rhs, emie.SolverConfig(tol=1e-6, restart=40, max_iters=500))
    ref = RE.reference_chain(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a, rhs, 1e-6)
    for i in range(2):
        assert reps[i].status == "converged"
        xr, xf = ref["_ref"]["x"][i], ref["_ref_fma"]["x"][i]
        env = np.linalg.norm(xf - xr) / np.linalg.norm(xr)
        err = np.linalg.norm(x[i] - xr) / np.linalg.norm(xr)
        print(f"cfg2 pol {'xy'[i]}: device {err:.2e} envelope {env:.2e} iterations {reps[i].iterations} "
              f"vs {int(ref['_ref']['iters'][i])} (fma build {int(ref['_ref_fma']['iters'][i])})")
        assert err <= max(4.0 * env, 1e-6), (err, env)
        assert abs(reps[i].iterations - int(ref["_ref"]["iters"][i])) <= 2


def test_cfg2_solver_on_reference_operator(torch_cuda):
    c, model, grid = _setup(2)
    rhs = _rhs(c)
    ref = RE.reference_chain(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a, rhs, 1e-8,
                             variants=("_ref",), want_blocks=True)["_ref"]
    op = emie.transform_operator(ref["blocks"], c.nx, c.ny, c.nz, c.omega)
    x, reps = emie.solve_cie(grid, model, op, rhs, emie.SolverConfig(tol=1e-8, restart=40, max_iters=500))
    for i in range(2):
        err = np.linalg.norm(x[i] - ref["x"][i]) / np.linalg.norm(ref["x"][i])
        assert reps[i].status == "converged"
        assert err <= 1e-7, err
        assert abs(reps[i].iterations - int(ref["iters"][i])) <= 1
