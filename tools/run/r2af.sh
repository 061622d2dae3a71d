set -u
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > gpurun_out/r2af_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/r2af_fuzz.log
