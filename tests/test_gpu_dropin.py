"""Drop-in evidence: the reference's own toeplitz suite
(/root/reference/proj/tests/test_toeplitz.cpp, unchanged) compiled against the
B200 C++ drop-in (include/emie/*.hpp over libemie_cu.so) passes on the GPU.
The binary is built in the CPU container by `make -C oracle dropin`."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "dropin_test_toeplitz"

pytestmark = pytest.mark.gpu


def test_reference_toeplitz_suite_on_b200(torch_cuda):
    if not BIN.exists():
        pytest.fail("oracle/_ref/dropin_test_toeplitz missing: run __graft_entry__.build() (make -C oracle dropin)")
    r = subprocess.run([str(BIN), "-ts=toeplitz"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "12 passed" in r.stdout, r.stdout


def test_dropin_fgmres_map_preconditioner_and_hook(torch_cuda):
    """fgmres(LinearMap) / solve_cie of the drop-in: the device Krylov solver
    over a host map, flexible right preconditioning, live on_iteration
    (tests/cpp/dropin_fgmres.cpp)."""
    b = ROOT / "oracle" / "_ref" / "dropin_fgmres"
    if not b.exists():
        pytest.fail("oracle/_ref/dropin_fgmres missing: run __graft_entry__.build() (make -C oracle dropin)")
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "dropin_fgmres ok" in r.stdout
