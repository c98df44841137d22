"""Receiver tensors vs whole-space brute cubature at depths around and inside
the source interval's z-range (the face-plane and inside-range integrands)."""
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import paper_1512_06126_b200 as emie
from test_gpu_receivers import wholespace_tensors
sigma, omega = 0.02, 2 * np.pi * 3.0
model = emie.LayeredModel([0.0], [sigma, sigma])
breaks = [0.0, 100.0, 250.0, 400.0]
grid = emie.make_grid(model, breaks, 3, 2, 150.0, 120.0, x0=-100.0, y0=-60.0)
np.set_printoptions(precision=2, linewidth=200)
for z in [-1e-3, 0.0, 1e-3, 50.0, 100.0, 175.0, 400.0, 401.0]:
    rec = (520.0, -260.0, z)
    try:
        got = emie.receiver_tensors(grid, model, omega, rec, 1, 1)
    except Exception as e:
        print(z, "rejected:", e)
        continue
    errs = []
    for k in range(3):
        GE, GH = wholespace_tensors(rec, ((50.0, 200.0), (60.0, 180.0), (breaks[k], breaks[k + 1])), sigma, omega,
                                    n=32, split=3)
        errs.append((np.max(np.abs(got[k, 0] - GE)) / np.max(np.abs(GE)), np.max(np.abs(got[k, 1] - GH)) / np.max(np.abs(GH))))
    print(f"z={z}: " + "  ".join(f"k{k}: E {e:.1e} H {h:.1e}" for k, (e, h) in enumerate(errs)))
