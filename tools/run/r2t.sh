set -u
timeout 900 python tools/pcie_trace.py --out-dir gpurun_out --tag r2 > gpurun_out/r2t_log.txt 2>&1; echo "rc=$?" >> gpurun_out/r2t_log.txt
ls -la gpurun_out/r2_pcie_trace.json >> gpurun_out/r2t_log.txt 2>&1
