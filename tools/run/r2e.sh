set -u
for v in 0 4; do echo "KC_K1_VARIANT=$v"; KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2; done > gpurun_out/r2e_k1probe.txt 2>&1
KC_K1_VARIANT=4 timeout 600 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider > gpurun_out/r2e_hash_v4.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_hash_v4.log
KC_K1_VARIANT=4 ncu --set full --clock-control none --import-source on -k regex:k1_hash -s 3 -c 1 -o gpurun_out/r2e_k1_c2_tma python tools/c2_k1_probe.py c2 > gpurun_out/r2e_k1ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2e_k1_c2_tma.ncu-rep > gpurun_out/r2e_k1_c2_tma_summary.txt 2>&1
