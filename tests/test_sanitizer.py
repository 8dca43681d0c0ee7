"""compute-sanitizer over every kernel: memcheck (out-of-bounds and
misaligned accesses, leaks), racecheck (shared-memory hazards), synccheck (illegal barrier use),
on small inputs of each kernel (scripts/sanitize_case.py, which also checks every result against
the oracle).  The kernels rely on benign relaxed races in GLOBAL memory (duplicate
discovery of a vertex at the same level writes the same distance); racecheck covers shared
memory only."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["sssp1", "sssp2", "narrow", "small", "ms64", "wcc", "wsssp", "part", "pack"]


def _run(tool, case, timeout=900):
    cmd = ["compute-sanitizer", "--tool", tool, "--error-exitcode", "99",
           "--print-limit", "20", sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py"),
           case]
    if tool == "racecheck":
        cmd[3:3] = ["--racecheck-report", "hazard"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    out = r.stdout + r.stderr
    return r.returncode, out


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool, case):
    if tool != "memcheck" and case == "sssp2":
        pytest.skip("the n > 2^22 case runs under memcheck only (racecheck time)")
    rc, out = _run(tool, case)
    tail = "\n".join(out.splitlines()[-30:])
    if rc != 0 and "closed on this pool" in out:
        # the GPU pool can disable compute-sanitizer (its wrapper then refuses every run); the
        # kernels keep their own checks (device-validated sources, oracle parity everywhere)
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert rc == 0, tail
    # memcheck / synccheck end with "ERROR SUMMARY: 0 errors"; racecheck with
    # "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert ("ERROR SUMMARY: 0 errors" in out or
            "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out), tail
    assert f"case ok: {case}" in out, tail
