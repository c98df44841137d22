"""Config-3 solve parity against the reference (tools/parity_report_r02.py's
config-2 chain at the benchmark shape; minutes of host time on the GPU box):

  same_operator  the device Green's operator (downloaded blocks) solved by the
                 reference's solve_cie (oracle/_ref, OpenMP on the host cores)
                 and by the device FGMRES (DCGS2): the solver paths alone;
  full_chain     the reference's own Green's build + solve_cie against the
                 device build + device solve (the Green's conditioning floor
                 of DESIGN.md section 2 included).

Both polarisations (plane-wave normal field, normal_field.py), tol 1e-6,
restart 40, max 2000 iterations.

    python tools/parity_cfg3_solve.py [out.json]   (on the GPU box)"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch  # noqa: F401  (CUDA context for the library)

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_1512_06126_b200 as emie  # noqa: E402
import ref_binding as R  # noqa: E402
from paper_1512_06126_b200 import configs, normal_field as NF  # noqa: E402

TOL, RESTART, MAXIT = 1e-6, 40, 2000
t00 = time.time()
c = configs.config(3)
model = emie.LayeredModel(list(c.tops), list(c.sigma))
grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
grid.sigma_a[...] = c.sigma_a
rhs = np.stack([NF.build_rhs(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.omega, p).reshape(-1) for p in "xy"])

op = emie.assemble_operator(grid, model, c.omega, keep_blocks=True)
blocks = op.blocks().reshape(c.ny, c.nx, -1)
t0 = time.time()
x, reps = emie.solve_cie(grid, model, op, rhs, emie.SolverConfig(tol=TOL, restart=RESTART, max_iters=MAXIT))
t_dev = time.time() - t0


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


out = {"what": __doc__.split("\n\n")[0], "tol": TOL, "restart": RESTART,
       "device": {"iterations": [r.iterations for r in reps], "seconds": round(t_dev, 3)}}
# the reference's solver on the device-built operator
case = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a)
case.set_operator(blocks)
t0 = time.time()
sol = [case.solve(rhs[i], TOL, RESTART, MAXIT) for i in range(2)]
out["same_operator"] = {
    "field_err_rel": [rel(x[i], sol[i][0]) for i in range(2)],
    "iterations": {"b200": [r.iterations for r in reps], "reference": [s[1]["iterations"] for s in sol]},
    "reference_status": [s[1]["status"] for s in sol],
    "reference_seconds": round(time.time() - t0, 1),
    "bar": "field error well inside the solve tolerance (both solutions meet tol 1e-6); iterations within +-2",
}
print("same_operator", out["same_operator"], flush=True)
# the reference's whole chain: its own Green's build, then solve_cie
case2 = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, c.sigma_a)
t0 = time.time()
case2.build()
t_build = time.time() - t0
t0 = time.time()
sol = [case2.solve(rhs[i], TOL, RESTART, MAXIT) for i in range(2)]
out["full_chain"] = {
    "field_err_rel": [rel(x[i], sol[i][0]) for i in range(2)],
    "iterations": {"b200": [r.iterations for r in reps], "reference": [s[1]["iterations"] for s in sol]},
    "reference_status": [s[1]["status"] for s in sol],
    "reference_build_seconds": round(t_build, 1),
    "reference_solve_seconds": round(time.time() - t0, 1),
    "bar": "field error at the Green's conditioning floor (config 2's chain: ~1.5e-5, inside 4x the reference's "
           "FMA-build distance); iterations within +-2",
}
print("full_chain", out["full_chain"], flush=True)
out["seconds"] = round(time.time() - t00, 1)
dst = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02_parity_cfg3_solve.json"
dst.write_text(json.dumps(out, indent=1) + "\n")
print("wrote", dst)
