set -u
for v in 0 3 0 3; do echo "KC_K1_VARIANT=$v"; KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3; KC_K1_VARIANT=$v python tools/c5_probe.py 1048576 1000 | cut -d' ' -f1-6; KC_K1_VARIANT=$v python tools/c5_probe.py 16777216 100 | cut -d' ' -f1-6; done > gpurun_out/r2y_ab.txt 2>&1
