"""The device's V-functions (the inputs of the Green's filter sums) against
the reference: layered.cpp:67-129 (layer states), 222-395 (interval packs,
factors, tables), 397-408 (v_functions), evaluated by the build's own device
code through emie_cu_vfunctions.

Well-conditioned quantities (V1 = i omega mu0 W00(unit) and V4 = W10(cond) /
sigma at every lambda; all of them at moderate lambda) are pinned at 1e-12 of
their maximum modulus — the level test_layered.cpp:277-401 pins the tables at.
The two sums the filter sums take, V1 + V3 and V2 + V5, cancel: V1 and V3
agree to 13 digits as lambda -> 0 and eta^2 W00d ~ 2h as lambda -> inf
(layered.cpp:305-315), so in any double evaluation they carry the rounding
of their summands. They are held to 1e-12 of the summands' moduli (the
backward-error view), and the cancellation factors are asserted so the test
documents where the reference's own blocks lose their digits."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1512_06126_b200 as emie
import ref_binding as R
from conftest import golden
from paper_1512_06126_b200 import configs

pytestmark = pytest.mark.gpu
MU0 = 1.2566370614359172e-06


def test_vfunctions_match_golden_tables(torch_cuda):
    """Device V-functions vs the reference's moment tables committed in
    tests/golden/tables.npz (three-layer model of test_layered.cpp:22-27)."""
    g = golden("tables")
    model = emie.LayeredModel(list(g["tops"]), list(g["sigma"]))
    br = g["breaks"]
    grid = emie.make_grid(model, list(br), 1, 1, 1.0, 1.0)
    sb = np.asarray(grid.sigma_b)[:, None]
    nz = len(br) - 1
    iu = np.triu_indices(nz)
    dev = emie.vfunctions(model, br, float(g["omega"]), g["lams"])
    iwmu = 1j * float(g["omega"]) * MU0
    for t in range(len(g["lams"])):
        tu, tc = g["T"][t, 0], g["T"][t, 1]  # (6, nz, nz): (0,0) (1,0) (0,1) (1,1) (2,0) (0,2)
        V1, V2, V3, V4, V5 = iwmu * tu[0], iwmu * tc[0], -tc[3] / sb, tc[1] / sb, tc[4] / sb
        for q, want, summands in ((0, V1, None), (1, V1 + V3, (V1, V3)), (2, V2 + V5, (V2, V5)), (3, V4, None)):
            d, w = (dev[t, q], want) if q == 3 else (dev[t, q][iu], want[iu])
            if summands is None:
                scale = np.max(np.abs(w))
            else:
                scale = np.max(np.abs(summands[0][iu]) + np.abs(summands[1][iu]))
            err = np.max(np.abs(d - w)) / scale
            assert err <= 1e-12, f"lambda {g['lams'][t]}: V-quantity {q} error {err:.2e}"


@pytest.mark.parametrize("k", [1, 3])
def test_vfunctions_match_reference_on_lattice(torch_cuda, k):
    """The full filter lattice lambda_m / R (R = 7 km) of configs 1 and 3."""
    c = configs.config(k)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
    lams = np.exp(np.arange(-250, 201) * 0.2 + 0.0964) / 7000.0
    dev = emie.vfunctions(model, c.breaks, c.omega, lams)
    case = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega)
    iu = np.triu_indices(c.nz)
    hmax = float(np.max(np.diff(c.breaks)))
    smin = float(np.min(np.abs(np.asarray(grid.sigma_b))))
    worst = np.zeros(4)
    canc = 0.0
    for t, lam in enumerate(lams):
        v = case.vfunctions(lam)
        V1, V2, V3, V4, V5 = v
        # W20d = eta^2 W00d - 2h: the summands of V5 are |V5| + 2h / |sigma|
        rows = ((V1, np.abs(V1)), (V1 + V3, np.abs(V1) + np.abs(V3)),
                (V2 + V5, np.abs(V2) + np.abs(V5) + 2.0 * hmax / smin), (V4, np.abs(V4)))
        for q, (w, s) in enumerate(rows):
            d, ww, ss = (dev[t, q], w, s) if q == 3 else (dev[t, q][iu], w[iu], s[iu])
            worst[q] = max(worst[q], np.max(np.abs(d - ww)) / np.max(ss))
        canc = max(canc, np.max(np.abs(np.diag(V1))) / np.max(np.abs(np.diag(V1 + V3))))
    assert np.all(worst <= 1e-12), f"cfg{k}: worst V-quantity errors {worst}"
    # where the reference's blocks lose their digits: V1 + V3 at small lambda
    assert canc > 1e10, canc
