set -u
timeout 1200 python -m pytest tests/test_gpu_diff.py tests/test_gpu_fused.py tests/test_gpu_plans.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2m_diff.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_diff.log
for i in 1 2; do KC_K2_CASES=c3_planted_bf16,c3_planted_f16,identical_bf16 python tools/k2_bench.py one; done > gpurun_out/r2m_k2_bench.txt 2>&1
