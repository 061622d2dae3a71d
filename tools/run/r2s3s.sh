set -u
# sub-wave ring with 2 x 4 KiB slices (KC_K1_VARIANT=12) vs 4 x 2 KiB (0)
KC_K1_VARIANT=12 timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fuzz.py -k "k1" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3s_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3s_parity.log
for v in 0 12 0 12; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2 --b2b
  for cell in "65536 1000" "1048576 100" "1048576 200"; do KC_K1_VARIANT=$v python tools/c5_probe.py $cell; done
done > gpurun_out/r2s3s_ab.txt 2>&1
