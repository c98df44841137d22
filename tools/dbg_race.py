"""Debug: octant contraction determinism / racecheck on a small symmetric operator.
    python tools/dbg_race.py N NZ REPS"""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
sys.path.insert(0, "/root/repo/oracle")
import paper_1512_06126_b200 as emie
from test_gpu_octant import _symmetric_blocks
n, nz, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
blocks = _symmetric_blocks(n, nz, 5)
sop = emie.transform_operator(blocks, n, n, nz)
assert emie.xy_symmetric(sop)
L = emie.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
nrhs = 2
E = sop.ex * sop.ey
g = torch.Generator(device="cuda").manual_seed(3)
S0 = torch.complex(torch.rand(nrhs * E * 3 * nz, device="cuda", dtype=torch.float64, generator=g),
                   torch.rand(nrhs * E * 3 * nz, device="cuda", dtype=torch.float64, generator=g))
ref = None
bad = 0
for r in range(reps):
    S = S0.clone()
    emie._check(L.emie_cu_contract_modes(sop.handle, ctypes.c_void_p(S.data_ptr()), nrhs, 0, sop.qx * sop.qy, st))
    torch.cuda.synchronize()
    if ref is None:
        ref = S
    elif not torch.equal(ref, S):
        bad += 1
print(f"n={n} nz={nz}: {bad} of {reps - 1} repeats differ")
