"""compute-sanitizer over every kernel of the path (SURVEY.md §5 "Race
detection / sanitizers"): memcheck (out-of-bounds and misaligned accesses,
including on the VMM mappings of a restore), racecheck (shared-memory hazards
in the cp.async rings of K1/K5/K6 and the element queue of K2) and synccheck
(barrier and warp-sync misuse).  The workload is tests/sanitize_worker.py, which
also checks every result against the oracle."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))


def _sanitizer() -> str:
    p = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(p):
        pytest.skip("compute-sanitizer not found")
    return p


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    from paper_2605_03208_b200 import build
    build.build()
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--print-limit", "20",
           sys.executable, os.path.join(HERE, "sanitize_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    out = p.stdout + p.stderr
    if "compute-sanitizer is closed" in out:
        # the GPU pool replaced compute-sanitizer with a stub after sanitizer runs left GPUs
        # needing a reset; the round-1/2 clean runs are kept in profiles/r*_sanitizer_*.txt
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert "sanitize workload ok" in out, out[-6000:]
    # The only tolerated reports are host API error returns of the kernarg-layout
    # probe: cuFuncGetParamInfo is called with increasing indices until it returns
    # CUDA_ERROR_INVALID_VALUE, which is how the driver API reports the parameter
    # count (CUDA 12.9 has no cuFuncGetParamCount).  Device-side errors: none.
    api = re.findall(r"Program hit (\S+) .* on CUDA API call to (\w+)", out)
    assert all(e == "CUDA_ERROR_INVALID_VALUE" and f == "cuFuncGetParamInfo" for e, f in api), api
    if tool == "racecheck":
        m = re.search(r"RACECHECK SUMMARY: (\d+) hazards displayed \((\d+) errors, (\d+) warnings\)", out)
        assert m and m.groups() == ("0", "0", "0"), out[-6000:]
    else:
        m = re.search(r"ERROR SUMMARY: (\d+) error", out)
        assert m and int(m.group(1)) == len(api), out[-6000:]
