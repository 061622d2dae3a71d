set -u
# K1 DRAM-lockstep diagnostic: CpA with warps started at 8 staggered chunk phases (KC_K1_VARIANT=8)
for v in "0 0" "8 11600" "8 5800" "0 0" "8 11600" "8 5800"; do
  set -- $v
  echo "KC_K1_VARIANT=$1 KC_K1_STAGGER_NS=$2"
  KC_K1_VARIANT=$1 KC_K1_STAGGER_NS=$2 python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$1 KC_K1_STAGGER_NS=$2 python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), round(k['K1_hash']['ms']*1e3), 'us', 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3l_ab.txt 2>&1
KC_K1_VARIANT=8 timeout 600 python -m pytest tests/test_gpu_hash.py -k "2gib" -m gpu -q -p no:cacheprovider > gpurun_out/r2s3l_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3l_parity.log
