set -u
probe() {
  python tools/c2_k1_probe.py c3
  python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
for v in 0 6 0 6; do echo "KC_K1_VARIANT=$v"; KC_K1_VARIANT=$v probe; done > gpurun_out/r2v_ab.txt 2>&1
export KC_K1_VARIANT=6
timeout 600 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider > gpurun_out/r2v_hash.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_hash.log
ncu --set full --clock-control none -k regex:k1_hash -s 3 -c 1 -o gpurun_out/r2v_k1_cpe python tools/c2_k1_probe.py c3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2v_k1_cpe.ncu-rep > gpurun_out/r2v_k1_cpe_summary.txt 2>&1
