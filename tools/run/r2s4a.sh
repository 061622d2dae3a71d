set -u
# kc_restore_dev_into: closure tests (incl. the in-place cycle test), then the bench latency block
timeout 1800 python -m pytest tests/test_gpu_closure.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s4a_closure.log 2>&1; echo "rc=$?" >> gpurun_out/r2s4a_closure.log
for i in 1 2; do
python bench.py --no-configs --no-e2e --no-cpu-baseline --no-fused --steps 3 --quiet | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['capture_replay']
for k in ('device','device_inplace','device_ipc'):
    v=c[k]; print(k, round(v['latency_s']*1e3,1) if 'latency_s' in v else v, {a:round(b*1e3,2) for a,b in v.get('stages_s',{}).items()}, v.get('validated_bit_exact'))
print('cold', round(c['device']['cold']['latency_s']*1e3,1), 'value', round(d['value']))"
done > gpurun_out/r2s4a_latency.txt 2>&1
