set -u
for v in 0 5 0 5; do echo "KC_K1_VARIANT=$v"; KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2; KC_K1_VARIANT=$v python tools/c5_probe.py 65536 1000; done > gpurun_out/r2q_k1s.txt 2>&1
KC_K1_VARIANT=5 timeout 600 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider > gpurun_out/r2q_hash_v5.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_hash_v5.log
