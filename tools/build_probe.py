import sys, time, ctypes
sys.path.insert(0, '/root/repo') if False else None
import os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
cfg = configs.config(3)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
emie.warmup(reserve_bytes=8 << 30)
op = emie.assemble_operator(grid, model, cfg.omega); del op; torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter(); model.validate(); grid.validate(model); t1 = time.perf_counter()
    op = emie.assemble_operator(grid, model, cfg.omega); torch.cuda.synchronize(); t2 = time.perf_counter()
    del op; torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"validate {1e3*(t1-t0):.2f} ms  build {1e3*(t2-t1):.2f} ms  free {1e3*(t3-t2):.2f} ms")
