"""Round-2 parity report: the device path against the reference itself
(oracle/_ref, compiled from the reference sources; its FMA-contracted build
oracle/_ref_fma and 1-ulp perturbed inputs give the reference's own
arithmetic envelope, oracle/ref_envelope.py). The numbers the -m gpu parity
tests assert, collected in one file:

  greens[cfg]    sampled blocks of configs 1-4 (tests/test_gpu_greens_parity.py
                 offsets): device error / block max, the per-block envelope,
                 their ratio (max, median), and the well-conditioned xz / yz
                 components' error;
  vfunctions     the build's V-functions on the config-3 filter lattice vs
                 the reference's (tests/test_gpu_vfunctions.py);
  apply_cfg3     apply(SystemOperator) and apply(SpectralOperator) on the
                 device-built config-3 operator vs the reference's applies;
  chain_cfg2     device Green's build + both plane-wave solves (tol 1e-6) vs
                 the reference's build + solve_cie: field error, the
                 reference's own FMA-build distance, iteration counts.

    python tools/parity_report_r02.py [out.json]   (on the GPU box)"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch  # noqa: F401  (CUDA context for the library)

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1512_06126_b200 as emie  # noqa: E402
import ref_binding as R  # noqa: E402
import ref_envelope as RE  # noqa: E402
from paper_1512_06126_b200 import configs, normal_field as NF  # noqa: E402
from test_gpu_greens_parity import _comp_slices, _offsets  # noqa: E402

out = {"what": __doc__.split("\n\n")[0]}
t00 = time.time()


def setup(k):
    c = configs.config(k)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
    grid.sigma_a[...] = c.sigma_a
    return c, model, grid


# ---- Green's blocks --------------------------------------------------------
out["greens"] = {}
for k in (1, 2, 3, 4):
    c, model, grid = setup(k)
    offs = np.array(_offsets(k, c.nx, c.ny))
    dev = emie.assemble_block(grid, model, c.omega, offs[:, 0], offs[:, 1])
    ref = RE.reference_blocks(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, offs)
    scale = np.max(np.abs(ref["ref"]), axis=1)
    env = RE.envelope(ref)
    err = np.max(np.abs(dev - ref["ref"]), axis=1) / scale
    ratio = err / env
    xz = max(float(np.max(np.max(np.abs(dev[:, sl] - ref["ref"][:, sl]), axis=1) / scale))
             for sl in _comp_slices(c.nz).values())
    out["greens"][f"cfg{k}"] = {
        "grid": [c.nx, c.ny, c.nz], "offsets": int(len(offs)),
        "err_over_block_max": {"max": float(err.max()), "median": float(np.median(err))},
        "reference_envelope": {"max": float(env.max()), "median": float(np.median(env))},
        "err_over_envelope": {"max": float(ratio.max()), "median": float(np.median(ratio))},
        "xz_yz_err_over_block_max": xz,
        "bar": "ratio <= 4 per block, median <= 3.5; xz / yz <= 1e-10",
    }
    print(k, out["greens"][f"cfg{k}"], flush=True)

# ---- V-functions on the config-3 lattice ------------------------------------
c, model, grid = setup(3)
lams = np.exp(np.arange(-250, 201) * 0.2 + 0.0964) / 7000.0
dev = emie.vfunctions(model, list(c.breaks), c.omega, lams)
case = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega)
iu = np.triu_indices(c.nz)
hmax = float(np.max(np.diff(c.breaks)))
smin = float(np.min(np.abs(np.asarray(grid.sigma_b))))
worst = np.zeros(4)
canc = 0.0
for t, lam in enumerate(lams):
    V1, V2, V3, V4, V5 = case.vfunctions(lam)
    rows = ((V1, np.abs(V1)), (V1 + V3, np.abs(V1) + np.abs(V3)),
            (V2 + V5, np.abs(V2) + np.abs(V5) + 2.0 * hmax / smin), (V4, np.abs(V4)))
    for q, (w, sm) in enumerate(rows):
        d, ww, ss = (dev[t, q], w, sm) if q == 3 else (dev[t, q][iu], w[iu], sm[iu])
        worst[q] = max(worst[q], float(np.max(np.abs(d - ww)) / np.max(ss)))
    canc = max(canc, float(np.max(np.abs(np.diag(V1))) / np.max(np.abs(np.diag(V1 + V3)))))
out["vfunctions_cfg3_lattice"] = {
    "lambdas": int(len(lams)),
    "max_err_over_summands": {"V1": worst[0], "V1+V3": worst[1], "V2+V5": worst[2], "V4": worst[3]},
    "V1_over_V1+V3_max": canc,
    "bar": "1e-12 of the summands' moduli (test_layered.cpp:277-401 pins the tables at this level)",
}
print(out["vfunctions_cfg3_lattice"], flush=True)

# ---- config-3 applies on the device-built operator ------------------------
op = emie.assemble_operator(grid, model, c.omega, keep_blocks=True)
blocks = op.blocks().reshape(c.ny, c.nx, -1)
refc = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a)
refc.set_operator(blocks)
sysop = emie.build_system(grid, op)
rng = np.random.default_rng(1234)
n = 3 * c.cells()
rec = {"octant_contraction": bool(emie.xy_symmetric(op))}
for which, dev_op in (("system", sysop), ("spectral", op)):
    errs = []
    for _ in range(2):
        u = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        want = refc.apply(which, u)
        errs.append(float(np.max(np.abs(emie.apply(dev_op, u) - want)) / np.max(np.abs(want))))
    rec[f"apply_{which}_max_rel"] = max(errs)
rec["bar"] = "1e-12 of max (test_toeplitz.cpp:314-325)"
out["apply_cfg3_device_built_operator"] = rec
print(rec, flush=True)

# ---- config-2 chain --------------------------------------------------------
c, model, grid = setup(2)
rhs = np.stack([NF.build_rhs(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.omega, p).reshape(-1) for p in "xy"])
op = emie.assemble_operator(grid, model, c.omega)
x, reps = emie.solve_cie(grid, model, op, rhs, emie.SolverConfig(tol=1e-6, restart=40, max_iters=500))
ref = RE.reference_chain(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a, rhs, 1e-6)
pol = {}
for i in range(2):
    xr, xf = ref["_ref"]["x"][i], ref["_ref_fma"]["x"][i]
    pol["xy"[i]] = {
        "field_err_rel": float(np.linalg.norm(x[i] - xr) / np.linalg.norm(xr)),
        "reference_fma_build_distance": float(np.linalg.norm(xf - xr) / np.linalg.norm(xr)),
        "iterations": {"b200": reps[i].iterations, "reference": int(ref["_ref"]["iters"][i]),
                       "reference_fma_build": int(ref["_ref_fma"]["iters"][i])},
    }
out["chain_cfg2_build_and_solve"] = {"tol": 1e-6, "polarisations": pol,
                                     "bar": "field error <= max(4 x the reference's FMA distance, 1e-6), "
                                            "iterations within +-2"}
print(out["chain_cfg2_build_and_solve"], flush=True)
out["seconds"] = round(time.time() - t00, 1)
dst = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02_parity_report.json"
dst.write_text(json.dumps(out, indent=1) + "\n")
print("wrote", dst)
