set -u
# restores reuse the physical allocations parked by released restores (KC_PHYS_PARK default on) vs off
timeout 2400 python -m pytest tests/test_gpu_closure.py tests/test_gpu_sequence.py tests/test_gpu_tracker.py tests/test_gpu_multi.py tests/test_gpu_host_ref.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3y_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3y_parity.log
for v in 1 0 1 0; do
  echo "KC_PHYS_PARK=$v"
  KC_PHYS_PARK=$v python bench.py --no-configs --no-e2e --no-cpu-baseline --no-fused --steps 3 --quiet | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['capture_replay']
for k in ('device','device_ipc','host_pinned'):
    v=c[k]; print(k, round(v['latency_s']*1e3,1), {a:round(b*1e3,2) for a,b in v['stages_s'].items()})
print('cold', round(c['device']['cold']['latency_s']*1e3,1))"
done > gpurun_out/r2s3y_ab.txt 2>&1
