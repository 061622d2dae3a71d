set -u
KC_K1_VARIANT=7 timeout 600 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider > gpurun_out/r2ab_hash_v7.log 2>&1; echo "rc=$?" >> gpurun_out/r2ab_hash_v7.log
for v in 0 7 0 7; do echo "KC_K1_VARIANT=$v"; KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2; KC_K1_VARIANT=$v python tools/c5_probe.py 65536 1000 | cut -d' ' -f1-6; done > gpurun_out/r2ab_ab.txt 2>&1
KC_K1_VARIANT=7 ncu --set full --clock-control none --import-source on -k regex:k1_hash -s 3 -c 1 -o gpurun_out/r2ab_k1_bulk python tools/c2_k1_probe.py c2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2ab_k1_bulk.ncu-rep > gpurun_out/r2ab_k1_bulk_summary.txt 2>&1
