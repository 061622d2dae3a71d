set -u
# where a small K2 launch spends its time: 64 KiB x 1k bytes pairs through the prepared plan
ncu --set full --clock-control none --import-source on -k regex:k2_diff -c 1 -o gpurun_out/r2s3v_k2_small python tools/c5_probe.py 65536 1000 > gpurun_out/r2s3v_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r2s3v_k2_small.ncu-rep > gpurun_out/r2s3v_k2_small_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_" --csv --log-file gpurun_out/r2s3v_launches.csv python tools/c5_probe.py 65536 1000 > gpurun_out/r2s3v_launch.log 2>&1
