set -u
# K1 ring shapes after the swizzled rows: 0 = CpA 8 warps x 3 x 1 KiB, 10 = 6 x 4, 11 = 4 x 6
KC_K1_VARIANT=10 timeout 600 python -m pytest tests/test_gpu_hash.py -k "2gib or many_small or edge" -m gpu -q -p no:cacheprovider > gpurun_out/r2s3r_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3r_parity.log
KC_K1_VARIANT=11 timeout 600 python -m pytest tests/test_gpu_hash.py -k "2gib or many_small or edge" -m gpu -q -p no:cacheprovider >> gpurun_out/r2s3r_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3r_parity.log
for v in 0 10 11 0 10 11; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3r_ab.txt 2>&1
