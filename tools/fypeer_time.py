"""Launch the fused forward y pass of the sharded apply (rank 1 of a G-rank
octant plan at config 3, all destinations local) a few times, for ncu
timing of the owner computation on the store path: python tools/fypeer_time.py G"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402
from paper_1512_06126_b200 import distributed as D  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = configs.config(3)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
sop = emie.assemble_operator(grid, model, cfg.omega)
nrhs = 2
plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G, octant=True)
rank = min(1, G - 1)
sh = D.cuda_shard(grid, sop, plan, rank, nrhs)
rng = np.random.default_rng(5)
U = torch.from_numpy(D.slab_of(rng.uniform(-1, 1, (nrhs, 3 * cfg.cells())) + 0j, plan, rank, nrhs)).cuda()
dsts = [torch.zeros((nrhs, plan.E, 3 * plan.nz), dtype=torch.complex128, device="cuda") for _ in range(G)]
assert sh.be.fused_peer_forward
for _ in range(4):
    sh.be.lateral_forward_peer(U, dsts, nrhs)
torch.cuda.synchronize()
print("ok")
