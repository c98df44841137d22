"""First vs warm device Green's builds of config 3 in one process:
    python tools/cold_build.py cold|warm [reserve_GB]
warm: library init (emie.warmup, optionally reserving reserve_GB in the pool) first."""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402

cfg = configs.config(3)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
torch.cuda.synchronize()
if sys.argv[1] == "warm":
    gb = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    t = time.perf_counter()
    emie.warmup(int(gb * (1 << 30)))
    torch.cuda.synchronize()
    print("init", time.perf_counter() - t)
for i in range(3):
    t = time.perf_counter()
    op = emie.assemble_operator(grid, model, cfg.omega)
    torch.cuda.synchronize()
    print(sys.argv[1], i, time.perf_counter() - t)
    del op
