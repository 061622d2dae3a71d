set -u
# K1 round formulations (probe) and the one-warp-per-SMSP sub-wave ring (KC_K1_VARIANT=7: kernel round, 8: late-add round)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/k1_round_probe tools/probes/k1_round_probe.cu && ./build/k1_round_probe > gpurun_out/r2s3c_probe.txt 2>&1
for v in 7 8; do
KC_K1_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fuzz.py -k "k1" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3c_parity_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3c_parity_$v.log
done
for v in 0 7 8 0 7 8; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2
  KC_K1_VARIANT=$v python tools/c5_probe.py 65536 1000
  KC_K1_VARIANT=$v python tools/c5_probe.py 1048576 100
done > gpurun_out/r2s3c_ab.txt 2>&1
KC_K1_VARIANT=8 ncu --set full --clock-control none --import-source on -k regex:k1_hash_ws -c 1 -o gpurun_out/r2s3c_ws8_c2 python tools/c2_k1_probe.py c2 > gpurun_out/r2s3c_ncu.log 2>&1
