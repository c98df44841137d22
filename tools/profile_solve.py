"""FGMRES on config 3's two plane-wave right-hand sides for ncu launch lists:
    python tools/profile_solve.py [--iters 40] [--config 3]"""
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
ap.add_argument("--iters", type=int, default=40)
a = ap.parse_args()
cfg = configs.config(a.config)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
sop = emie.assemble_operator(grid, model, cfg.omega)
sysop = emie.build_system(grid, sop)
rhs = np.stack([NF.build_rhs(cfg.tops, cfg.sigma, cfg.breaks, cfg.nx, cfg.ny, cfg.omega, p).reshape(-1)
                for p in ("x", "y")])
d = torch.from_numpy(rhs.reshape(-1)).cuda()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, reps = emie.fgmres_system(sysop, d, emie.SolverConfig(tol=1e-6, restart=40, max_iters=a.iters))
    torch.cuda.synchronize()
    print(f"solve {rep}: {time.perf_counter() - t0:.4f} s, iterations {[r.iterations for r in reps]}")
