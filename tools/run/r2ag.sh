set -u
timeout 900 python -m pytest tests/test_gpu_host_ref.py tests/test_gpu_sanitizer.py -m gpu -q -p no:cacheprovider -k "host_ref or memcheck" > gpurun_out/r2ag_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ag_tests.log
