set -u
# session-3 re-entry: confirm the restored tree on the GPU (build, smoke, tests, bench)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s3a_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s3a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s3a_pytest.log
timeout 900 python bench.py > gpurun_out/r2s3a_bench.json 2> gpurun_out/r2s3a_bench.err; echo "bench rc=$?" >> gpurun_out/r2s3a_bench.err
