set -u
# small closures (c1, c2 configs) with the restore park on / off / on for spans >= 64 MiB only
for v in "1 0" "0 0" "1 67108864" "1 0" "0 0" "1 67108864"; do
  set -- $v
  echo "KC_PHYS_PARK=$1 KC_PHYS_PARK_MIN=$2"
  KC_PHYS_PARK=$1 KC_PHYS_PARK_MIN=$2 python bench.py --no-e2e --no-cpu-baseline --no-fused --steps 3 --quiet | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['configs']; cr=d['capture_replay']
for k in ('c1','c2'):
    v=c[k]['closure']['device']; print(k, round(v['latency_s']*1e3,2), 'restore', round(v['restore_s']*1e3,2))
print('c4 device', round(cr['device']['latency_s']*1e3,1), 'restore', round(cr['device']['stages_s']['restore_total']*1e3,1), 'inplace', round(cr['device_inplace']['latency_s']*1e3,1))"
done > gpurun_out/r2s4c_ab.txt 2>&1
