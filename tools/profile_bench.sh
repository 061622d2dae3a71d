#!/bin/bash
# Reproduce the profiles/ evidence for the bench step (run on the B200 box, one GPU):
#   launch list (per-launch times, cold-cache, serialised) and one ncu --set full
#   capture of each step kernel (K1 post-manifest, K2 bf16 pool-pair diff, K5 fused).
# Outputs go to gpurun_out/; tools/ncu_summary.py turns the .ncu-rep files into text.
set -u
O=${1:-gpurun_out}
mkdir -p "$O"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-latency --no-configs --no-cpu-baseline"
[ "${SKIP_LIST:-0}" = 1 ] || ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|k5_|kc_fixture" --csv \
    --log-file "$O/launches.csv" $B --no-fused > "$O/launch_run.log" 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k2_diff<.int.10," \
    --launch-skip 1 -c 1 -o "$O/k2_bench" $B --no-fused > "$O/k2_ncu.log" 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"CpCfg<.int.8, .int.3, .int.1024, .bool.1>, .bool.0>" --launch-skip 3 -c 1 -o "$O/k1_bench" $B --no-fused \
    > "$O/k1_ncu.log" 2>&1
[ "${SKIP_K5:-0}" = 1 ] || ncu --set full --clock-control none --import-source on -k regex:k5_hash_cmp -c 1 -o "$O/k5_bench" $B \
    > "$O/k5_ncu.log" 2>&1
for r in k2_bench k1_bench k5_bench; do
    [ -f "$O/$r.ncu-rep" ] && python tools/ncu_summary.py "$O/$r.ncu-rep" > "$O/${r}_summary.txt" 2>&1
done
