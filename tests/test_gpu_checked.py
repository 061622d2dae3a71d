"""The bounds-checked build (libkc_checked.so, -DKC_CHECKS=1) under the oracle-checked
workloads.  The GPU pool has compute-sanitizer disabled (tests/test_gpu_sanitizer.py
skips there), so this is the memory-safety evidence for the kernels added since its
last clean run (the warp-specialized sub-wave K1 ring, the swizzled ring rows): every
cp.async into a ring slot, every shared read of a slice, every K2 queue push and every
chunk -> region lookup is checked on the device and traps with the failing condition.
The workloads compare every result with the oracle, so a clean run is also correct."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def checked_env():
    from paper_2605_03208_b200 import build
    build.build()
    lib = build.build_lib(checked=True)
    env = dict(os.environ, KC_LIB="checked")
    out = subprocess.run([sys.executable, "-c", "from paper_2605_03208_b200 import kc; kc.lib(); print(kc.LIB_PATH)"],
                         env=env, capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.stdout.strip() == lib, out.stdout + out.stderr
    return env


def _run(cmd, env, timeout):
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=ROOT, timeout=timeout)
    out = p.stdout + p.stderr
    assert "KC_DCHECK failed" not in out, out[-6000:]
    return p.returncode, out


def test_checked_build_sanitizer_workload(checked_env):
    """Every kernel of the path (K1 sub-wave ring / CpS / CpA / generic, K3, digests, K2 every
    dtype family, K5 + filtered K2, K6 capture and restore, replay, validate) on the checked
    build, each result against the oracle."""
    rc, out = _run([sys.executable, os.path.join(HERE, "sanitize_worker.py")], checked_env, 1800)
    assert rc == 0 and "sanitize workload ok" in out, out[-6000:]


def test_checked_build_k1_and_k2_parity(checked_env):
    """The K1 edge, boundary and randomized region-set parity tests and the 600 random K2
    cases on the checked build."""
    rc, out = _run([sys.executable, "-m", "pytest", "tests/test_gpu_hash.py", "tests/test_gpu_fuzz.py", "-m", "gpu",
                    "-q", "-x", "-p", "no:cacheprovider"], checked_env, 2400)
    assert rc == 0, out[-6000:]
