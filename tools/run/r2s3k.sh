set -u
# K1: the warp-specialized ring at every size (KC_K1_VARIANT=7: 3 hashing warps alone on SMSPs 0-2, 24 chunks/SM) vs the cp.async ring (0)
KC_K1_VARIANT=7 timeout 900 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3k_parity_7.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3k_parity_7.log
for v in 0 7 0 7; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3k_ab.txt 2>&1
