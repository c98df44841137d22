"""Time repeated device Green's builds of config 3 (cold vs warm)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import time, torch, numpy as np
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
cfg = configs.config(3)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    sop = emie.assemble_operator(grid, model, 2 * np.pi * cfg.freqs[0])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("build", i, round(t1 - t0, 4))
    del sop
    torch.cuda.synchronize()
