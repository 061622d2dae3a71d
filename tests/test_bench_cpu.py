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


def test_reference_arm_runs_on_cpu_with_our_config():
    """--impl reference times the CPU oracle (no GPU needed) and prints the same metric,
    unit and config as our arm, with a cpu_baseline describing the run and an e2e object."""
    sys.path.insert(0, ROOT)
    import bench
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--ref-step-seconds", "0.1", "--cpu-sample-mb", "12"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["impl"] == "reference" and r["metric"] == bench.METRIC and r["unit"] == bench.UNIT
    assert r["config"] == bench.workload_config(1)
    cb = r["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == (os.cpu_count() or 1) and cb["value"] == r["value"] > 0
    assert cb["hash_gbs"] > 0 and cb["diff_gbs"] > 0 and cb["host"]["nproc"] == os.cpu_count()
    assert r["e2e"] == {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_c4_host_sample_is_stratified_and_bounded():
    """The oracle's c4 sample takes the head of every one of the 185 regions (every region
    kind), in whole chunks, within the requested size."""
    sys.path.insert(0, ROOT)
    import bench
    s = bench.c4_sample(None, 24)
    assert len(s) == 185
    assert all(r.size == a.size and r.size % 2 == 0 for r, a, _ in s)
    assert sum(r.size for r, _, _ in s) <= 24 * 2**20 + 185 * 65536
    assert {dt for _, _, dt in s} == {bench.DTC["bf16"], bench.DTC["u64"], bench.DTC["i32"], bench.DTC["f32"]}


def test_oracle_rates_are_bounded_and_consistent():
    """bench_configs.oracle_rates: the oracle on host threads over (ref, act, dtype) pairs;
    max_bytes keeps only the first pieces, and the step mix is 4N / (2N/H + 2N/D)."""
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench_configs as bc
    rng = np.random.default_rng(0)
    pairs = [(rng.integers(0, 256, 6 << 20, dtype=np.uint8), None, 0)]
    pairs = [(r, r.copy(), 0) for r, _, _ in pairs]
    r1 = bc.oracle_rates(pairs, 2, 0.0)
    assert r1["bytes"] == 6 << 20 and r1["hash_gbs"] > 0 and r1["diff_gbs"] > 0
    H, D = r1["hash_gbs"], r1["diff_gbs"]
    assert abs(r1["step_mix_gbs"] - 4 / (2 / H + 2 / D)) < 1e-9 * r1["step_mix_gbs"]
    r2 = bc.oracle_rates(pairs, 1, 0.0, max_bytes=bc.PIECE)
    assert r2["bytes"] == bc.PIECE
    info = bc.host_info()
    assert info["nproc"] == (os.cpu_count() or 1)


def test_profile_renderers_on_committed_evidence():
    """tools/baseline_table.py and tools/pcie_trace.py --summarize re-derive BASELINE.md's
    table and the PCIe summary from the committed round-2 evidence (no GPU)."""
    b = os.path.join(ROOT, "profiles", "r2_bench_n1.json")
    t = os.path.join(ROOT, "profiles", "r2_pcie_trace.json")
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "tools", "baseline_table.py"), b], text=True)
    assert "| c4 30 GB MoE pool, N = 1 |" in out and out.count("| c5 ") == 6
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "tools", "pcie_trace.py"), "--summarize", t,
                                   "57.2", "55.6"], text=True)
    rows = {ln.split()[0]: ln.split() for ln in out.splitlines() if ln[:3] in ("D2H", "H2D")}
    assert int(rows["D2H"][6].replace(",", "")) == int(rows["H2D"][6].replace(",", "")) > 29_000_000_000
