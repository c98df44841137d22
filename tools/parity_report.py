"""Parity report: B200 path vs the reference's golden outputs (tests/golden).
Writes a JSON summary (default profiles/parity_report.json)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1512_06126_b200 as emie  # noqa: E402

out = {}
for name in ["toeplitz_single", "toeplitz_tiny", "toeplitz_small", "toeplitz_large", "cfg1"]:
    g = dict(np.load(ROOT / "tests" / "golden" / f"{name}.npz"))
    nx, ny, nz = int(g["nx"]), int(g["ny"]), len(g["breaks"]) - 1
    rec = {"grid": [nx, ny, nz]}
    sop = emie.transform_operator(g["blocks"], nx, ny, nz, float(g["omega"]))
    spec = np.concatenate(sop.comp)
    rec["spectra_rel"] = float(np.max(np.abs(spec - g["spec"])) / np.max(np.abs(g["spec"])))
    rec["applyB_rel"] = max(float(np.max(np.abs(emie.apply(sop, v) - w)) / np.max(np.abs(w)))
                            for v, w in zip(g["vecs"], g["applyB"]))
    model = emie.LayeredModel(list(g["tops"]), list(g["sigma"]))
    grid = emie.make_grid(model, list(g["breaks"]), nx, ny, float(g["hx"]), float(g["hy"]))
    grid.sigma_a[...] = g["sigma_a"].reshape(grid.sigma_a.shape)
    sys_op = emie.build_system(grid, sop)
    rec["applyA_rel"] = max(float(np.max(np.abs(emie.apply(sys_op, v) - w)) / np.max(np.abs(w)))
                            for v, w in zip(g["vecs"], g["applyA"]))
    dev = emie.assemble_operator(grid, model, float(g["omega"]), keep_blocks=True)
    b = dev.blocks()
    rec["greens_block_rel_max"] = float(max(np.max(np.abs(b[i, j] - g["blocks"][i, j])) / np.max(np.abs(g["blocks"][i, j]))
                                            for i in range(ny) for j in range(nx)))
    if name == "cfg1":
        x, reps = emie.solve_cie(grid, model, sop, g["rhs"], emie.SolverConfig(tol=1e-10))
        rec["solve_tol1e-10_rel"] = [float(np.linalg.norm(x[i] - g["x_tol10"][i]) / np.linalg.norm(g["x_tol10"][i])) for i in range(2)]
        x6, reps6 = emie.solve_cie(grid, model, sop, g["rhs"], emie.SolverConfig(tol=1e-6))
        rec["solve_tol1e-6_rel"] = [float(np.linalg.norm(x6[i] - g["x_tol6"][i]) / np.linalg.norm(g["x_tol6"][i])) for i in range(2)]
        rec["iterations_tol1e-6"] = {"b200": [r.iterations for r in reps6], "reference": [int(v) for v in g["iters_tol6"]]}
        # solve with the device-built operator (Green's build + solve, end to end)
        xd, repd = emie.solve_cie(grid, model, dev, g["rhs"], emie.SolverConfig(tol=1e-6))
        rec["solve_device_greens_tol1e-6_rel"] = [float(np.linalg.norm(xd[i] - g["x_tol6"][i]) / np.linalg.norm(g["x_tol6"][i])) for i in range(2)]
    out[name] = rec
    print(name, json.dumps(rec))
dst = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "parity_report.json"
dst.write_text(json.dumps(out, indent=1))
