"""bench.py host logic that needs no GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_world_mismatch_fails_fast():
    """--gpus N under a launcher that started a different number of ranks is an error,
    never a silently mislabelled 1-GPU number."""
    e = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=e, cwd=ROOT)
    assert p.returncode == 2
    assert "WORLD_SIZE" in json.loads(p.stdout.strip().splitlines()[-1])["error"]
