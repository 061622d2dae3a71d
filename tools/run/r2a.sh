set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 600 python bench.py --gpus 2 > gpurun_out/r2a_bench_n2.json 2> gpurun_out/r2a_bench_n2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err
