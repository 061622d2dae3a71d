set -u
# K1 warp-specialized sub-wave ring (KC_K1_VARIANT=4) vs the cp.async ring (0): parity, c2 and c5 timings; op latencies
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/op_latency tools/probes/op_latency.cu && ./build/op_latency > gpurun_out/r2s3b_oplat.txt 2>&1
KC_K1_VARIANT=4 timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fuzz.py -k "k1" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3b_parity.log
for v in 0 4 0 4; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2
  KC_K1_VARIANT=$v python tools/c5_probe.py 65536 1000
  KC_K1_VARIANT=$v python tools/c5_probe.py 4096 100000
done > gpurun_out/r2s3b_ab.txt 2>&1
KC_K1_VARIANT=4 ncu --set full --clock-control none --import-source on -k regex:k1_hash_ws -c 1 -o gpurun_out/r2s3b_ws_c2 python tools/c2_k1_probe.py c2 > gpurun_out/r2s3b_ncu.log 2>&1
for v in 0 5 6 0 5 6; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3b_large.txt 2>&1
KC_K1_VARIANT=5 timeout 600 python -m pytest tests/test_gpu_hash.py -k "2gib or many_small" -m gpu -q -p no:cacheprovider > gpurun_out/r2s3b_parity_large.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3b_parity_large.log
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_sequence.py tests/test_gpu_tracker.py -m gpu -q -p no:cacheprovider > gpurun_out/r2s3b_rest.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3b_rest.log
