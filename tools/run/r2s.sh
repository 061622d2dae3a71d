set -u
ncu --set full --clock-control none --import-source on -k regex:k1_hash -s 3 -c 1 -o gpurun_out/r2s_k1_c2 python tools/c2_k1_probe.py c2 > gpurun_out/r2s_k1ncu.log 2>&1
ncu -i gpurun_out/r2s_k1_c2.ncu-rep --page source --csv > gpurun_out/r2s_k1_c2_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/r2s_k1_c2.ncu-rep > gpurun_out/r2s_k1_c2_summary.txt 2>&1
