set -u
timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fused.py -m gpu -q -p no:cacheprovider > gpurun_out/r2r_hash.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_hash.log
for i in 1 2; do for c in c2 c3; do python tools/c2_k1_probe.py $c; done; python tools/c5_probe.py 65536 1000; done > gpurun_out/r2r_k1.txt 2>&1
python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'fused', round(d['fused_step']['K5_plus_filtered_K2']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/r2r_k1.txt 2>&1
