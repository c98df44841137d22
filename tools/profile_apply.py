"""Short cfg3 apply loop for ncu / nsight captures (one GPU):
    python tools/profile_apply.py [--config 3] [--applies 3] [--greens]"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=3)
p.add_argument("--applies", type=int, default=3)
p.add_argument("--nrhs", type=int, default=2)
a = p.parse_args()
cfg = configs.config(a.config)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
sop = emie.assemble_operator(grid, model, cfg.omega)
sys_op = emie.build_system(grid, sop)
n = 3 * cfg.cells()
U = torch.randn(a.nrhs * n, dtype=torch.complex128, device="cuda")
for _ in range(a.applies):
    W = emie.apply(sys_op, U)
torch.cuda.synchronize()
print("ok", float(W.abs().max()))
