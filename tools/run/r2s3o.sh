set -u
# after the swizzled rows: K1 ring configs re-ranked (0 = CpA 64 chunks x 3 x 1 KiB, 3 = CpD 128 x 3 x 512 B), bench-step profiles incl. K5
for v in 0 3 0 3; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --no-fused --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3o_ab.txt 2>&1
timeout 1500 bash tools/profile_bench.sh gpurun_out/r2s3o_prof > gpurun_out/r2s3o_prof.log 2>&1; echo "prof rc=$?" >> gpurun_out/r2s3o_prof.log
