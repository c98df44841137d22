import sys, numpy as np
sys.path.insert(0, '.')
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
from paper_1512_06126_b200.sharding import shard_indices
cfg = configs.config(3); freqs = configs.config(5).freqs
print("rank freqs N=8:", [shard_indices(len(freqs), 8, r)[0] for r in range(8)])
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
bad = []
for i, f in enumerate(freqs):
    try:
        sop = emie.assemble_operator(grid, model, 2 * np.pi * f)
        sys_ = emie.build_system(grid, sop)
        v = np.ones(3 * cfg.cells(), np.complex128)
        w = emie.apply(sys_, v)
        ok = np.all(np.isfinite(w))
        if not ok: bad.append((i, f, "nonfinite"))
    except Exception as e:
        bad.append((i, f, repr(e)[:120]))
print("bad:", bad)
