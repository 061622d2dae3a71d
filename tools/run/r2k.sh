set -u
for c in "65536 1000" "4096 100000"; do
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --csv --clock-control none -k regex:"k1_|k2_|memset|k3_" python tools/c5_probe.py $c > gpurun_out/r2k_c5_$(echo $c | tr ' ' _).csv 2>&1
  python tools/c5_probe.py $c >> gpurun_out/r2k_c5_times.txt 2>&1
done
