set -u
timeout 1200 python -m pytest tests/test_gpu_diff.py tests/test_gpu_plans.py tests/test_gpu_host_ref.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_tests.log
for u in 1 0 1 0; do echo "KC_K2_SMALL_U4=$u"; KC_K2_SMALL_U4=$u python tools/c5_probe.py 65536 1000; KC_K2_SMALL_U4=$u python tools/c5_probe.py 1048576 100; done > gpurun_out/r2u_ab.txt 2>&1
