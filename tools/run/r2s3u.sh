set -u
# K2 with 4 KiB units for small launches (default) vs 16 KiB everywhere (KC_K2_SMALL_UNITS=0)
timeout 1800 python -m pytest tests/test_gpu_diff.py tests/test_gpu_fuzz.py tests/test_gpu_fused.py tests/test_gpu_host_ref.py tests/test_gpu_plans.py tests/test_gpu_closure.py tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3u_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3u_parity.log
for v in 1 0 1 0; do
  echo "KC_K2_SMALL_UNITS=$v"
  for cell in "65536 1000" "1048576 100" "4096 10000" "4096 100000" "65536 2000" "16384 1000"; do KC_K2_SMALL_UNITS=$v python tools/c5_probe.py $cell; done
done > gpurun_out/r2s3u_ab.txt 2>&1
