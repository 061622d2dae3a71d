set -u
free -g > gpurun_out/r2b_host.txt; nproc >> gpurun_out/r2b_host.txt; lscpu >> gpurun_out/r2b_host.txt
for c in c2 c3; do python tools/c2_k1_probe.py $c; done > gpurun_out/r2b_k1probe.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
