set -u
# final validation of the round's last tree: smoke, all GPU tests, bench defaults, reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s4b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s4b_smoke.log
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2s4b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s4b_pytest.log
timeout 900 python bench.py > gpurun_out/r2s4b_bench.json 2> gpurun_out/r2s4b_bench.err; echo "bench rc=$?" >> gpurun_out/r2s4b_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2s4b_ref.json 2> gpurun_out/r2s4b_ref.err; echo "ref rc=$?" >> gpurun_out/r2s4b_ref.err
