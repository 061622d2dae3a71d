"""A9 / E on CUDA: the N > 1 bench path through the CUDA kernels.

``bench.py --gpus 2`` launches two ranks itself (torch.distributed.run on
127.0.0.1).  On a one-GPU box both ranks share cuda:0 and the collectives run
over gloo (KC_BENCH_ONE_GPU=1, KC_BENCH_BACKEND=gloo): every byte is still
hashed and diffed by libkc.so's kernels, each rank over its E1 shard of the
30 GB c4 pool, and the C2/C3/C4 results of the timed step are combined.  O7
(SURVEY.md 8(c)): the combined post-manifest, finalized reports and per-region
bitmaps must equal the 1-GPU run's bit for bit.  The reference pool is planted
with 1-byte mismatches (--plant) so reports and bitmaps are not trivially
zero.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

ARGS = ["--steps", "2", "--warmup", "1", "--no-e2e", "--no-fused", "--no-latency", "--no-cpu-baseline", "--no-configs", "--plant",
        "--quiet"]


def _bench(n, env=None, extra=()):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), *ARGS, *extra],
                       capture_output=True, text=True, timeout=900, env=e, cwd=ROOT)
    assert p.returncode == 0, f"bench --gpus {n} failed:\n{p.stdout[-3000:]}\n{p.stderr[-3000:]}"
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout        # rank 0 alone prints
    return json.loads(lines[0])


@pytest.fixture(scope="module")
def one():
    return _bench(1)


KEYS = ("post_manifest_sha256_excl_ptr_tables", "reports_sha256", "bitmaps_sha256", "bitmap_bits", "chunks",
        "report_counter_sums", "max_ulp", "max_abs", "max_rel")


@pytest.mark.parametrize("placement,combine", [("e1", "nccl"), ("e2", "nccl"), ("e1", "peer")])
def test_n2_one_gpu_combine_equals_n1(one, placement, combine):
    """E1: each rank its own regions.  E2: rank 0 owns the whole pool and rank 1
    hashes/diffs half of its chunks through a kc_peer_import mapping of rank 0's
    allocations (on one GPU a second mapping of the same HBM; over NVLink on two).
    combine=peer: no data collective -- each rank's K1 stores its post-manifest, and
    its K2 its reports and bitmap bits, into its slice of rank 0's buffers through
    peer mappings; rank 0 reads the combined results from its own HBM."""
    two = _bench(2, {"KC_BENCH_ONE_GPU": "1", "KC_BENCH_BACKEND": "gloo"},
                 ["--placement", placement, "--combine", combine])
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["collectives"]["backend"] == "gloo"
    f1, f2 = one["fingerprint"], two["fingerprint"]
    assert f1["report_counter_sums"][0] > 0 and f1["bitmap_bits"] > 0 and f1["max_ulp"] > 0   # planted
    for k in KEYS:
        assert f1[k] == f2[k], (k, f1[k], f2[k])
    assert two["gpu_launches"] > 0 and "A9_combine_ms" in two["kernels"]


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or __import__("torch").cuda.device_count() < 2,
                    reason="needs two GPUs (NCCL over NVLink)")
@pytest.mark.parametrize("placement", ["e1", "e2"])
def test_n2_nccl_two_gpus_equals_n1(one, placement):
    two = _bench(2, extra=["--placement", placement])
    assert two["n_gpus"] == 2 and two["collectives"]["backend"] == "nccl"
    for k in KEYS:
        assert one["fingerprint"][k] == two["fingerprint"][k], k
