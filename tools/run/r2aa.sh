set -u
for u in 1 0 1 0; do echo "KC_K2_SMALL_U4=$u"; for c in "4096 100000" "4096 10000" "65536 10000"; do KC_K2_SMALL_U4=$u python tools/c5_probe.py $c; done; done > gpurun_out/r2aa_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_diff.py tests/test_gpu_plans.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2aa_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2aa_tests.log
