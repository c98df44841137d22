"""The reference's own quad suite (/root/reference/proj/tests/test_quad.cpp,
unchanged) compiled against the drop-in's include/emie/quad.hpp and
bessel_zeros (paper_1512_06126_b200/cpp/emie_quad.cpp): host-side quadrature
utilities of the reference API (test and oracle machinery, no device work),
so this runs in the CPU tier. Built by `make -C oracle dropin`."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "dropin_test_quad"


def test_reference_quad_suite_against_dropin():
    if not BIN.exists():
        pytest.skip("oracle/_ref/dropin_test_quad not built (no /root/reference here)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "8 passed" in r.stdout and "0 failed" in r.stdout, r.stdout
