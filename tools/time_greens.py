"""Time repeated device Green's builds of a config (wall time and the library's
own CUDA-event stage timers: 5 = assemble kernel, 6 = spectra transform).
    python tools/time_greens.py [--config 3] [--reps 3]"""
import argparse
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = configs.config(a.config)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
L = emie.lib()
L.emie_cu_profile_enable.argtypes = [ctypes.c_int]
L.emie_cu_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
ms = np.zeros(8)
cnt = np.zeros(8, np.int64)
torch.cuda.synchronize()
for i in range(a.reps):
    L.emie_cu_profile_collect(ms.ctypes.data, cnt.ctypes.data, 8)
    L.emie_cu_profile_enable(1)
    t0 = time.perf_counter()
    sop = emie.assemble_operator(grid, model, 2 * np.pi * cfg.freqs[0])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    L.emie_cu_profile_enable(0)
    L.emie_cu_profile_collect(ms.ctypes.data, cnt.ctypes.data, 8)
    print(f"build {i}: wall {t1 - t0:.4f} s  assemble {ms[5]:.1f} ms  spectra {ms[6]:.1f} ms")
    del sop
    torch.cuda.synchronize()
