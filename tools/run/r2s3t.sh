set -u
# end-of-round validation after the swizzled ring rows: smoke, GPU tests, bench (defaults), reference arm, launch list
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3t_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s3t_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r2s3t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s3t_pytest.log
timeout 900 python bench.py > gpurun_out/r2s3t_bench.json 2> gpurun_out/r2s3t_bench.err; echo "bench rc=$?" >> gpurun_out/r2s3t_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2s3t_ref.json 2> gpurun_out/r2s3t_ref.err; echo "ref rc=$?" >> gpurun_out/r2s3t_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|k5_|kc_fixture" --csv --log-file gpurun_out/r2s3t_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-latency --no-configs --no-cpu-baseline --no-fused > gpurun_out/r2s3t_launch_run.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2s3t_launch_run.log
