"""Device Green's build of a config for ncu: python tools/profile_greens.py [--config 1]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=1)
a = p.parse_args()
cfg = configs.config(a.config)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
sop = emie.assemble_operator(grid, model, cfg.omega)
print("ok", sop.ex)
