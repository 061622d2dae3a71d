set -u
timeout 900 python -m pytest tests/test_gpu_hash.py tests/test_gpu_fused.py -m gpu -q -p no:cacheprovider > gpurun_out/r2d_hash.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_hash.log
for c in c2 c3; do python tools/c2_k1_probe.py $c; done > gpurun_out/r2d_k1probe.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_hash -s 3 -c 1 -o gpurun_out/r2d_k1_c2 python tools/c2_k1_probe.py c2 > gpurun_out/r2d_k1ncu.log 2>&1
ncu -i gpurun_out/r2d_k1_c2.ncu-rep --page source --csv > gpurun_out/r2d_k1_c2_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2d_k1_c2.ncu-rep > gpurun_out/r2d_k1_c2_summary.txt 2>&1
