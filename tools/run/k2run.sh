set -x
python -m pytest tests/test_gpu_diff.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
for q in 0 1; do KC_K2_Q2=$q python tools/k2_bench.py one; done
