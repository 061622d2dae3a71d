set -u
# last-tree confirmation: smoke, closure / hash / checked-build tests
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s4d_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s4d_smoke.log
timeout 1800 python -m pytest tests/test_gpu_closure.py tests/test_gpu_hash.py tests/test_gpu_checked.py -m gpu -q -p no:cacheprovider > gpurun_out/r2s4d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s4d_pytest.log
