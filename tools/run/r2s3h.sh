set -u
# default K1 now routes <= 4 x SMs groups through the warp-specialized ring; KC_K1_VARIANT=4 = round-2 sub-wave path
timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fuzz.py tests/test_gpu_plans.py tests/test_gpu_fused.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3h_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3h_parity.log
for v in 0 4 0 4; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2 --b2b
  for cell in "65536 1000" "1048576 100" "1048576 160" "1048576 256" "65536 4000"; do KC_K1_VARIANT=$v python tools/c5_probe.py $cell; done
done > gpurun_out/r2s3h_ab.txt 2>&1
