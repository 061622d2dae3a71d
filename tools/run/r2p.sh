set -u
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_smoke.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tests/sanitize_worker.py > gpurun_out/r2p_sanitizer_$t.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2p_ref.json 2> gpurun_out/r2p_ref.err
