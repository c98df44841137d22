"""Device V-functions (emie_cu_vfunctions) vs the reference's v_functions
along the filter lattice (GPU box). Prints, per lambda, the worst relative
error of V1, V1+V3, V2+V5, V4 (upper triangle; V4 full) against each
quantity's max modulus, and the cancellation factor |V1|/|V1+V3| that
explains where V1+V3 loses digits in any double-precision evaluation.

    python tools/vfunc_probe.py 1 3
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_1512_06126_b200 as emie  # noqa: E402
import ref_binding as R  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402


def run(k, radius):
    c = configs.config(k)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    lams = np.exp(np.arange(-250, 201) * 0.2 + 0.0964) / radius
    dev = emie.vfunctions(model, c.breaks, c.omega, lams)
    case = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega)
    nz = c.nz
    iu = np.triu_indices(nz)
    rows = []
    for t, lam in enumerate(lams):
        v = case.vfunctions(lam)
        want = [v[0], v[0] + v[2], v[1] + v[4], v[3]]
        errs = []
        for q in range(4):
            w = want[q] if q == 3 else want[q][iu]
            d = dev[t, q] if q == 3 else dev[t, q][iu]
            errs.append(np.max(np.abs(d - w)) / max(np.max(np.abs(w)), 1e-300))
        canc = np.max(np.abs(np.diag(v[0]))) / max(np.max(np.abs(np.diag(v[0] + v[2]))), 1e-300)
        rows.append((lam, *errs, canc))
    rows = np.array(rows)
    np.save(ROOT / "gpurun_out" / f"vfunc_cfg{k}_R{int(radius)}.npy", rows)
    print(f"cfg{k} R={radius}: worst relative errors over 451 lambdas "
          f"V1 {rows[:,1].max():.1e} V13 {rows[:,2].max():.1e} V25 {rows[:,3].max():.1e} V4 {rows[:,4].max():.1e}")
    for r in rows[::25]:
        print(f"  lam {r[0]:.2e}: V1 {r[1]:.1e} V13 {r[2]:.1e} V25 {r[3]:.1e} V4 {r[4]:.1e}  |V1|/|V1+V3| {r[5]:.1e}")
    return rows


if __name__ == "__main__":
    for a in sys.argv[1:] or ["1"]:
        run(int(a), 7000.0)
