set -u
timeout 1800 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2z_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_multi.log
KC_BENCH_ONE_GPU=1 KC_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 2 --no-e2e --no-latency --no-configs --combine peer > gpurun_out/r2z_peer.json 2> gpurun_out/r2z_peer.err
