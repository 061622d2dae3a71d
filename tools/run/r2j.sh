set -u
timeout 1200 python -m pytest tests/test_gpu_plans.py tests/test_gpu_hash.py tests/test_gpu_fused.py tests/test_gpu_host_ref.py -m gpu -q -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
for c in c2 c3; do python tools/c2_k1_probe.py $c; done > gpurun_out/r2j_k1probe.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_hash -s 3 -c 1 -o gpurun_out/r2j_k1_c2 python tools/c2_k1_probe.py c2 > gpurun_out/r2j_k1ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2j_k1_c2.ncu-rep > gpurun_out/r2j_k1_c2_summary.txt 2>&1
timeout 900 python bench.py --no-latency --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
