"""Break down the host-buffer apply (e2e) of config 3: pipelined call, single-rhs call, device applies, copies."""
import sys, time, ctypes
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
cfg = configs.config(3)
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
sop = emie.assemble_operator(grid, model, cfg.omega)
sysop = emie.build_system(grid, sop)
L = emie.lib()
n = 3 * cfg.cells()
hin = torch.empty(2 * n, dtype=torch.complex128).pin_memory(); hin.copy_(torch.randn(2*n, dtype=torch.complex128))
hout = torch.empty(2 * n, dtype=torch.complex128).pin_memory()
st = torch.cuda.current_stream(); sp = ctypes.c_void_p(st.cuda_stream)
d = torch.empty(2*n, dtype=torch.complex128, device='cuda'); o = torch.empty_like(d)
def t(fn, k=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
print("host apply nrhs=2 (pipelined) ms", t(lambda: L.emie_cu_apply_system_host(sysop.handle, ctypes.c_void_p(hin.data_ptr()), ctypes.c_void_p(hout.data_ptr()), 2, sp)))
print("host apply nrhs=1 ms", t(lambda: L.emie_cu_apply_system_host(sysop.handle, ctypes.c_void_p(hin.data_ptr()), ctypes.c_void_p(hout.data_ptr()), 1, sp)))
print("device apply nrhs=1 ms", t(lambda: L.emie_cu_apply_system(sysop.handle, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(o.data_ptr()), 1, sp)))
print("device apply nrhs=2 ms", t(lambda: L.emie_cu_apply_system(sysop.handle, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(o.data_ptr()), 2, sp)))
h1 = hin[:n]; d1 = d[:n]
print("H2D 25MB ms", t(lambda: d1.copy_(h1, non_blocking=True)))
print("D2H 25MB ms", t(lambda: h1.copy_(d1, non_blocking=True)))
