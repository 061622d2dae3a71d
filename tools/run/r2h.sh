set -u
for q in 2 3 4 2 3 4; do echo "KC_K2_Q2=$q"; KC_K2_CASES=c3_planted_bf16,c3_planted_f16,identical_bf16 KC_K2_Q2=$q python tools/k2_bench.py one; done > gpurun_out/r2h_k2_bench.txt 2>&1
