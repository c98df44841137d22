"""FGMRES convergence of the plane-wave solves of a config (device path):
iterations, final relative residual and the residual every 100 iterations.
    python tools/solve_convergence.py [--config 3] [--max-iters 4000] [--restart 40] [--freq F]"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402
from paper_1512_06126_b200 import normal_field as NF  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--max-iters", type=int, default=4000)
ap.add_argument("--restart", type=int, default=40)
ap.add_argument("--freq", type=float, default=None)
a = ap.parse_args()
cfg = configs.config(a.config)
freq = a.freq if a.freq is not None else cfg.freqs[0]
omega = 2 * np.pi * freq
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
sop = emie.assemble_operator(grid, model, omega)
sysop = emie.build_system(grid, sop)
rhs = np.stack([NF.build_rhs(cfg.tops, cfg.sigma, cfg.breaks, cfg.nx, cfg.ny, omega, p).reshape(-1)
                for p in ("x", "y")])
d = torch.from_numpy(rhs.reshape(-1)).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
_, reps = emie.fgmres_system(sysop, d, emie.SolverConfig(tol=1e-6, restart=a.restart, max_iters=a.max_iters))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
for p, r in zip("xy", reps):
    h = np.asarray(r.history)
    print(f"cfg{a.config} f={freq:g} Hz pol {p}: {r.status} after {r.iterations} iterations, residual {r.residual:.3e}, "
          f"{dt:.2f} s; every 100: {' '.join(f'{v:.1e}' for v in h[::100])}")
