set -u
probe() {
  python tools/c2_k1_probe.py c3
  python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for v in 0 3 0 3; do echo "KC_K1_VARIANT=$v"; KC_K1_VARIANT=$v probe; done > gpurun_out/r2aj_ab.txt 2>&1
