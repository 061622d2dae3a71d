export KC_K2_CASES=c3_planted_bf16
ncu --set full --clock-control none --import-source on -k regex:k2_diff --launch-skip 3 -c 1 -o gpurun_out/k2_planted python tools/k2_bench.py one > gpurun_out/k2ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/k2_planted.ncu-rep > gpurun_out/k2_planted_summary.txt 2>&1
python tools/ncu_sass_hist.py gpurun_out/k2_planted.ncu-rep >> gpurun_out/k2_planted_summary.txt 2>&1
