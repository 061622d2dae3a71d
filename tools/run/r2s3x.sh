set -u
# the bounds-checked build under the oracle-checked workloads; then the full GPU suite on the default build
timeout 2400 python -m pytest tests/test_gpu_checked.py -m gpu -q -p no:cacheprovider > gpurun_out/r2s3x_checked.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3x_checked.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_checked.py > gpurun_out/r2s3x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s3x_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3x_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s3x_smoke.log
timeout 900 python bench.py > gpurun_out/r2s3x_bench.json 2> gpurun_out/r2s3x_bench.err; echo "bench rc=$?" >> gpurun_out/r2s3x_bench.err
