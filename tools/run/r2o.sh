set -u
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_host_ref.py tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
