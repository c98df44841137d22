"""GPU FGMRES parity: solve_cie on config 1 against the reference's own
solve (tests/golden/cfg1.npz), plus the SPEC.md:381-384 properties."""
import numpy as np
import pytest

import paper_1512_06126_b200 as emie
from conftest import golden

pytestmark = pytest.mark.gpu


def _cfg1():
    g = golden("cfg1")
    nz = len(g["breaks"]) - 1
    sop = emie.transform_operator(g["blocks"], int(g["nx"]), int(g["ny"]), nz, float(g["omega"]))
    model = emie.LayeredModel(list(g["tops"]), list(g["sigma"]))
    grid = emie.make_grid(model, list(g["breaks"]), int(g["nx"]), int(g["ny"]), float(g["hx"]), float(g["hy"]))
    grid.sigma_a[...] = g["sigma_a"].reshape(grid.sigma_a.shape)
    return g, model, grid, sop


def test_solve_matches_reference_cfg1(torch_cuda):
    g, model, grid, sop = _cfg1()
    # both polarisations in one lockstep solve
    x, reps = emie.solve_cie(grid, model, sop, g["rhs"], emie.SolverConfig(tol=1e-10))
    for i in range(2):
        assert reps[i].status == "converged"
        want = g["x_tol10"][i]
        assert np.linalg.norm(x[i] - want) <= 1e-8 * np.linalg.norm(want)
    x6, reps6 = emie.solve_cie(grid, model, sop, g["rhs"], emie.SolverConfig(tol=1e-6))
    for i in range(2):
        assert reps6[i].status == "converged"
        assert abs(reps6[i].iterations - int(g["iters_tol6"][i])) <= 1
        want = g["x_tol6"][i]
        # fields E_n = U_n / a_n share a per-cell factor: compare U directly
        assert np.linalg.norm(x6[i] - want) <= 1e-6 * np.linalg.norm(want)
        h = np.array(reps6[i].history)
        assert np.all(np.diff(h[: min(40, len(h))]) <= 1e-12)  # monotone inside a cycle


def test_zero_rhs_and_identity(torch_cuda):
    g, model, grid, sop = _cfg1()
    n = g["rhs"].shape[1]
    x, reps = emie.solve_cie(grid, model, sop, np.zeros(n, np.complex128), emie.SolverConfig(tol=1e-8))
    assert reps[0].status == "converged" and reps[0].iterations == 0 and np.all(x == 0)
    # zero contrast: A = identity, converges in one iteration with U = rhs
    grid0 = emie.make_grid(model, list(g["breaks"]), int(g["nx"]), int(g["ny"]), float(g["hx"]), float(g["hy"]))
    x, reps = emie.solve_cie(grid0, model, sop, g["rhs"][0], emie.SolverConfig(tol=1e-8))
    assert reps[0].status == "converged" and reps[0].iterations == 1
    assert np.max(np.abs(x - g["rhs"][0])) <= 1e-14 * np.max(np.abs(g["rhs"][0]))


def test_bad_config(torch_cuda):
    g, model, grid, sop = _cfg1()
    with pytest.raises(emie.InvalidArgument):
        emie.solve_cie(grid, model, sop, g["rhs"][0], emie.SolverConfig(tol=0.0))


def _odd_system(nx, ny, nz, scale, seed):
    rng = np.random.default_rng(seed)
    nent = 2 * nz * (2 * nz + 1)
    blocks = scale * (rng.standard_normal((ny, nx, nent)) + 1j * rng.standard_normal((ny, nx, nent)))
    sop = emie.transform_operator(blocks, nx, ny, nz)
    model = emie.LayeredModel([0.0, 5000.0], [0.0, 0.01, 0.1])
    breaks = list(np.linspace(10.0, 10.0 + 50.0 * nz, nz + 1))
    grid = emie.make_grid(model, breaks, nx, ny, 100.0, 120.0)
    grid.sigma_a[...] = 10.0 ** rng.uniform(-3, 0, grid.sigma_a.shape)
    n = 3 * nx * ny * nz
    b = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
    return sop, emie.build_system(grid, sop), b


@pytest.mark.parametrize("nx,ny,nz,restart", [(5, 3, 3, 40), (7, 4, 8, 12), (16, 3, 8, 40)])
def test_solve_residual_odd_sizes(torch_cuda, nx, ny, nz, restart):
    """field lengths that are not a multiple of the CGS2 tile (128 entries):
    the returned solution's true residual, through the independently checked
    apply, meets the tolerance"""
    sop, sys, b = _odd_system(nx, ny, nz, 1e-3, nx * 100 + restart)
    x, reps = emie.fgmres_system(sys, b, emie.SolverConfig(tol=1e-9, restart=restart, max_iters=400))
    for i in range(2):
        assert reps[i].status == "converged"
        r = emie.apply(sys, x[i]) - b[i]
        assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(b[i])


def test_long_cycle_untiled_fallback(torch_cuda):
    """a 60-vector cycle: steps past the tiled sweeps' 41 staged vectors run
    the untiled CGS2 kernels; the Givens residual estimate still tracks the
    true residual (orthogonality kept across the switch)"""
    sop, sys, b = _odd_system(6, 5, 4, 0.2, 77)
    x, reps = emie.fgmres_system(sys, b, emie.SolverConfig(tol=1e-15, restart=60, max_iters=55))
    for i in range(2):
        assert reps[i].iterations == 55
        true = np.linalg.norm(emie.apply(sys, x[i]) - b[i]) / np.linalg.norm(b[i])
        assert abs(true - reps[i].residual) <= 1e-9 + 1e-6 * true
        assert abs(reps[i].history[54] - true) <= 1e-8 + 1e-4 * true


def test_fgmres_over_python_map_hook_and_preconditioner(torch_cuda):
    """fgmres(LinearMap) (cie.hpp:71-72) over a Python callable: the device
    Krylov iteration with host callbacks reproduces the system solve; the
    hook runs live with the history; right preconditioning converges;
    exceptions raised by the map come back unchanged."""
    g, model, grid, sop = _cfg1()
    sysop = emie.build_system(grid, sop)
    b = g["rhs"][0]
    cfg = emie.SolverConfig(tol=1e-10, restart=12)
    xs, reps = emie.fgmres_system(sysop, b, cfg)
    seen, calls = [], [0]

    def A(u):
        calls[0] += 1
        return emie.apply_host(sysop, u)

    x, rep = emie.fgmres(A, b, emie.SolverConfig(tol=1e-10, restart=12, on_iteration=lambda i, r: seen.append((i, r))))
    assert rep.status == "converged" and rep.iterations == reps[0].iterations
    assert np.max(np.abs(x - xs)) <= 1e-13 * np.max(np.abs(xs))
    assert [i for i, _ in seen] == list(range(1, rep.iterations + 1))
    assert [r for _, r in seen] == rep.history
    assert calls[0] == rep.iterations + -(-rep.iterations // 12)  # + one residual per cycle, no speculation
    # flexible right preconditioning (z_j = M v_j, x += sum y_j z_j): with M a
    # scaling the Krylov space is unchanged, so the iterates match the plain solve
    xp, rp = emie.fgmres(A, b, emie.SolverConfig(tol=1e-10, restart=12, right_precond=lambda v: 0.5 * v))
    assert rp.status == "converged" and rp.iterations == rep.iterations, (rp.iterations, rp.residual)
    assert np.max(np.abs(xp - xs)) <= 1e-9 * np.max(np.abs(xs))
    r = b - emie.apply_host(sysop, xp)
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b)

    def boom(u):
        raise KeyError("map failed")
    with pytest.raises(KeyError):
        emie.fgmres(boom, b, emie.SolverConfig(tol=1e-8))
    # the system solve's hook (device vectors, two right-hand sides in lockstep)
    seen2 = []
    _, reps2 = emie.fgmres_system(sysop, g["rhs"], emie.SolverConfig(tol=1e-6, on_iteration=lambda k, i, r: seen2.append((k, i, r))))
    for k in range(2):
        assert [r for kk, _, r in seen2 if kk == k] == reps2[k].history


def _solve_in_subprocess(dcgs2, restart, max_iters, tol, precond=False):
    """the library reads EMIE_CU_DCGS2 once per process"""
    import os
    import subprocess
    import sys
    import tempfile
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = f"""
import numpy as np, sys
sys.path.insert(0, {str(root)!r}); sys.path.insert(0, {str(root / 'tests')!r})
import paper_1512_06126_b200 as emie
from test_gpu_solve import _odd_system
sop, sysop, b = _odd_system(7, 4, 8, 0.2, 31)
cfg = emie.SolverConfig(tol={tol}, restart={restart}, max_iters={max_iters})
if {precond}:  # flexible right preconditioning over host callbacks, one rhs per solve
    cfg.right_precond = lambda v: 0.5 * v
    out = [emie.fgmres(lambda u: emie.apply_host(sysop, u), b[i], cfg) for i in range(2)]
    x, reps = np.stack([o[0] for o in out]), [o[1] for o in out]
else:
    x, reps = emie.fgmres_system(sysop, b, cfg)
res = [np.linalg.norm(emie.apply(sysop, x[i]) - b[i]) / np.linalg.norm(b[i]) for i in range(2)]
np.savez(sys.argv[1], x=x, it=[r.iterations for r in reps], est=[r.residual for r in reps], res=res,
         h=np.array(reps[0].history))
"""
    with tempfile.NamedTemporaryFile(suffix=".npz", delete=False) as f:
        out = f.name
    env = dict(os.environ, EMIE_CU_DCGS2="1" if dcgs2 else "0")
    subprocess.run([sys.executable, "-c", code, out], env=env, check=True)
    return dict(np.load(out))


@pytest.mark.parametrize("restart,max_iters,tol,precond",
                         [(40, 400, 1e-10, False), (7, 300, 1e-9, False), (12, 200, 1e-9, True), (40, 23, 1e-14, False)])
def test_dcgs2_matches_cgs2(torch_cuda, restart, max_iters, tol, precond):
    """DCGS2 (one dots sweep and one update sweep per step; v_j's second
    projection delayed into the next step, the Hessenberg column corrected
    and re-rotated on the host, the solution's coefficients mapped back to
    the corrected basis) against CGS2: the same Krylov iterates in exact
    arithmetic, so equal iteration counts (+-1), solutions to the solve's
    tolerance, and a residual estimate that tracks the true residual -- also
    when the solve stops inside a cycle (max_iters 23) and with a flexible
    right preconditioner (the Z basis)"""
    a = _solve_in_subprocess(True, restart, max_iters, tol, precond)
    b = _solve_in_subprocess(False, restart, max_iters, tol, precond)
    for i in range(2):
        assert abs(int(a["it"][i]) - int(b["it"][i])) <= 1
        assert np.linalg.norm(a["x"][i] - b["x"][i]) <= 1e3 * tol * np.linalg.norm(b["x"][i])
        assert abs(a["res"][i] - a["est"][i]) <= 1e-9 + 1e-3 * a["res"][i]
        if max_iters > 100:
            assert a["res"][i] <= 2 * tol
