"""compute-sanitizer over small solves (tools/sanitize_case.py): memcheck
(out-of-bounds and misaligned accesses, including the 16-byte / 8-byte
aligned word loads at arena ends), racecheck and synccheck (shared memory
and barriers), with normal hashes and with PO_DEBUG_HASH_BITS=3 (every
dictionary insert collides: concurrent claims, publish/verify races between
warps, the byte-verified fix-up). SURVEY.md §5."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("bits", [None, 3])
def test_compute_sanitizer_clean(tool, bits):
    if not Path(SAN).exists():
        pytest.skip("compute-sanitizer not found")
    env = dict(os.environ)
    env.pop("PO_DEBUG_HASH_BITS", None)
    if bits:
        env["PO_DEBUG_HASH_BITS"] = str(bits)
    rows = "1500" if tool == "racecheck" else "3000"
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=99", "--target-processes=all",
           sys.executable, str(ROOT / "tools" / "sanitize_case.py"), rows]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, env=env)
    out = r.stdout + r.stderr
    print(out[-3000:])
    if r.returncode == 86 and "closed on this pool" in out:
        # the pool's wrapper refuses the tool (it is not a result about this
        # code); the round-2 runs before the closure were clean
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case ok" in out
    # memcheck / synccheck: "ERROR SUMMARY: 0 errors"; racecheck: "RACECHECK
    # SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards displayed (0 errors" in out
