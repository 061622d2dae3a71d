set -u
# K1 register-fed (KC_K1_VARIANT=5: 512 thr x 1 CTA/SM, 6: 512 x 2) vs the cp.async ring (0) on the pool and c3
for v in 5 6; do
KC_K1_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3j_parity_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3j_parity_$v.log
done
for v in 0 5 6 0 5 6; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3j_ab.txt 2>&1
