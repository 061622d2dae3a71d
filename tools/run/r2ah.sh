set -u
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/r2ah_smi.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2ah_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ah_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ah_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2ah_smoke.log
timeout 900 python bench.py > gpurun_out/r2ah_bench.json 2> gpurun_out/r2ah_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2ah_ref.json 2> gpurun_out/r2ah_ref.err
