set -u
timeout 1200 python -m pytest tests/test_gpu_diff.py tests/test_gpu_fused.py tests/test_gpu_host_ref.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2f_diff.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_diff.log
for q in 1 2; do echo "KC_K2_Q2=$q"; KC_K2_Q2=$q python tools/k2_bench.py one; done > gpurun_out/r2f_k2_bench.txt 2>&1
export KC_K2_CASES=c3_planted_bf16
ncu --set full --clock-control none --import-source on -k regex:k2_diff --launch-skip 3 -c 1 -o gpurun_out/r2f_k2_planted python tools/k2_bench.py one > gpurun_out/r2f_k2ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2f_k2_planted.ncu-rep > gpurun_out/r2f_k2_planted_summary.txt 2>&1
python tools/ncu_sass_hist.py gpurun_out/r2f_k2_planted.ncu-rep >> gpurun_out/r2f_k2_planted_summary.txt 2>&1
