set -u
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i_pytest.log
python tools/k2_bench.py > gpurun_out/r2i_k2_bench.txt 2>&1
for q in 0 1 2 3; do echo "KC_K2_Q2=$q"; KC_K2_CASES=c3_planted_bf16,c3_planted_f16 KC_K2_Q2=$q python tools/k2_bench.py one; done > gpurun_out/r2i_k2_q2.txt 2>&1
export KC_K2_CASES=c3_planted_bf16
ncu --set full --clock-control none --import-source on -k regex:k2_diff --launch-skip 3 -c 1 -o gpurun_out/r2i_k2_planted python tools/k2_bench.py one > gpurun_out/r2i_k2ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2i_k2_planted.ncu-rep > gpurun_out/r2i_k2_planted_summary.txt 2>&1
python tools/ncu_sass_hist.py gpurun_out/r2i_k2_planted.ncu-rep >> gpurun_out/r2i_k2_planted_summary.txt 2>&1
unset KC_K2_CASES
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
