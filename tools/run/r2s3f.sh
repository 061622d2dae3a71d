set -u
# sub-wave K1: flush-between-calls vs back-to-back timing, variants 0 / 7 / 8
for v in 0 7 8 0 7 8; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2 --b2b
done > gpurun_out/r2s3f_ab.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv >> gpurun_out/r2s3f_ab.txt
