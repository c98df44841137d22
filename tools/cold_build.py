import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
cfg = configs.config(3)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
torch.cuda.synchronize()
if sys.argv[1] == "warm":
    t = time.perf_counter(); emie.warmup(); torch.cuda.synchronize(); print("init", time.perf_counter() - t)
for i in range(3):
    t = time.perf_counter(); op = emie.assemble_operator(grid, model, cfg.omega); torch.cuda.synchronize(); print(sys.argv[1], i, time.perf_counter() - t); del op
