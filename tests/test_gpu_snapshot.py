"""EMG1 operator snapshots (reference greens.cpp:373-446,
test_greens.cpp:289-348) through the B200 drop-in: an operator built on the
device round-trips bit for bit and foreign files are rejected
(tests/cpp/dropin_snapshot.cpp), the reference's own load_operator reads our
file to the same values, and its save_operator writes the same bytes back."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "dropin_snapshot"
TOOL = ROOT / "oracle" / "_ref" / "emie_ref_tool"

pytestmark = pytest.mark.gpu


def test_snapshot_roundtrip_and_reference_compat(torch_cuda, tmp_path):
    for b in (BIN, TOOL):
        if not b.exists():
            pytest.fail(f"{b} missing: run __graft_entry__.build()")
    r = subprocess.run([str(BIN), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    ours = json.loads(r.stdout.strip().splitlines()[-1])
    assert ours["failures"] == 0
    resaved = tmp_path / "resaved.bin"
    q = subprocess.run([str(TOOL), "snapshot-check", ours["path"], str(resaved)], capture_output=True,
                       text=True, timeout=300)
    assert q.returncode == 0, q.stdout + q.stderr
    ref = json.loads(q.stdout.strip().splitlines()[-1])
    assert ref["loaded"]
    for k in ("nx", "ny", "nz", "omega", "checksum"):
        assert ref[k] == ours[k], k
    assert Path(ours["path"]).read_bytes() == resaved.read_bytes()
