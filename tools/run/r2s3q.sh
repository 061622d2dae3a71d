set -u
# K2 with a bulk L2 prefetch of the warp's next unit (KC_K2_L2_PREFETCH=1) vs without
KC_K2_L2_PREFETCH=1 timeout 900 python -m pytest tests/test_gpu_diff.py tests/test_gpu_fuzz.py -k "not k1" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3q_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3q_parity.log
for v in 0 1 0 1; do
  echo "KC_K2_L2_PREFETCH=$v"
  KC_K2_L2_PREFETCH=$v python tools/k2_bench.py
  KC_K2_L2_PREFETCH=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  KC_K2_L2_PREFETCH=$v python tools/c5_probe.py 65536 1000
  KC_K2_L2_PREFETCH=$v python tools/c5_probe.py 1048576 1000
done > gpurun_out/r2s3q_ab.txt 2>&1
