"""Debug: host-buffer applies (emie_cu_apply_system_host) against the device apply, field by field.
    python tools/dbg_stream.py CONFIG K"""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
cfgid = int(sys.argv[1]); K = int(sys.argv[2])
cfg = configs.config(cfgid)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
sop = emie.assemble_operator(grid, model, cfg.omega)
sysop = emie.build_system(grid, sop)
n = 3 * cfg.cells()
rng = np.random.default_rng(1)
V = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
dev = emie.apply(sysop, torch.from_numpy(V.reshape(-1)).cuda()).cpu().numpy().reshape(2, n)
dev2 = emie.apply(sysop, torch.from_numpy(V.reshape(-1)).cuda()).cpu().numpy().reshape(2, n)
print("device repeat identical", np.array_equal(dev, dev2))
d1 = [emie.apply(sysop, torch.from_numpy(V[i]).cuda()).cpu().numpy() for i in range(2)]
print("device nrhs=1 vs batched", [np.array_equal(d1[i], dev[i]) for i in range(2)])
for rep in range(3):
    one = emie.apply_host(sysop, V).reshape(2, n)
    print("host call", rep, [float(np.max(np.abs(one[i] - d1[i]))) for i in range(2)])
big = np.tile(V, (K, 1))
out = emie.apply_host(sysop, big).reshape(2 * K, n)
print("streamed diffs", [float(np.max(np.abs(out[i] - d1[i % 2]))) for i in range(2 * K)])
