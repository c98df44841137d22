"""The oracle build of the reference passes the reference's own test suites
(pins the FFTW/Boost/doctest shims and the cie.cpp compile fix)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
FAST = ROOT / "oracle" / "_ref" / "emie_ref_fast_tests"


@pytest.fixture(scope="module")
def ref_tests():
    import sys
    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_binding
    ref_binding.build()
    if not FAST.exists():
        pytest.skip("oracle/_ref not built (no /root/reference and no prebuilt oracle)")
    return FAST


@pytest.mark.parametrize("suite", ["layered", "quad", "hankel", "toeplitz"])
def test_reference_suite_passes(ref_tests, suite):
    r = subprocess.run([str(ref_tests), f"-ts={suite}"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
