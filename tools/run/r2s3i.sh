set -u
# bench defaults after the sub-wave K1 ring and the write+read L2 flush of the config timer
timeout 900 python bench.py > gpurun_out/r2s3i_bench.json 2> gpurun_out/r2s3i_bench.err; echo "bench rc=$?" >> gpurun_out/r2s3i_bench.err
for v in 0 4; do
  echo "KC_K1_VARIANT=$v"
  for cell in "65536 1000" "1048576 100" "1048576 256" "65536 4000"; do KC_K1_VARIANT=$v python tools/c5_probe.py $cell; done
done > gpurun_out/r2s3i_c5.txt 2>&1
