set -u
# ncu --set full of the bench-step K1 (swizzled rows) and the c2 sub-wave ring
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-latency --no-configs --no-cpu-baseline --no-fused"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"CpCfg<.int.8, .int.3, .int.1024, .bool.1>, .bool.0>" --launch-skip 3 -c 1 -o gpurun_out/r2s3p_k1_bench $B > gpurun_out/r2s3p_k1_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2s3p_k1_bench.ncu-rep > gpurun_out/r2s3p_k1_bench_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_hash_ws -c 1 -o gpurun_out/r2s3p_ws_c2 python tools/c2_k1_probe.py c2 > gpurun_out/r2s3p_ws_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2s3p_ws_c2.ncu-rep > gpurun_out/r2s3p_ws_c2_summary.txt 2>&1
