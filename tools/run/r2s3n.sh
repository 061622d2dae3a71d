set -u
# K1/K5/K6 swizzled ring rows (each 128-byte global line fills one shared row) vs round 2's padded slices (K1: KC_K1_VARIANT=9)
timeout 1500 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fuzz.py tests/test_gpu_closure.py tests/test_gpu_plans.py tests/test_gpu_fused.py tests/test_gpu_host_ref.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3n_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3n_parity.log
for v in 0 9 0 9; do
  echo "KC_K1_VARIANT=$v"
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c3
  KC_K1_VARIANT=$v python tools/c2_k1_probe.py c2 --b2b
  KC_K1_VARIANT=$v python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; f=d.get('fused_step') or {}; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'fused', json.dumps(f)[:400], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done > gpurun_out/r2s3n_ab.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed_op_ldgsts.sum -k regex:k1_hash -c 2 python tools/c2_k1_probe.py c3 > gpurun_out/r2s3n_ncu_c3.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed_op_ldgsts.sum -k regex:k1_hash -c 2 python tools/c2_k1_probe.py c2 > gpurun_out/r2s3n_ncu_c2.txt 2>&1
