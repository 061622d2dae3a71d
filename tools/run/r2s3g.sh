set -u
for v in 0 7 0 7; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2 --flushes
done > gpurun_out/r2s3g_ab.txt 2>&1
