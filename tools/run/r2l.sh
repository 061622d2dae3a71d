set -u
bash tools/profile_bench.sh gpurun_out/r2l
