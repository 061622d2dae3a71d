set -u
# end-of-round validation after the sub-wave K1 ring: GPU tests, smoke, bench (defaults), reference arm, bench-step profiles
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3m_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s3m_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r2s3m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s3m_pytest.log
timeout 900 python bench.py > gpurun_out/r2s3m_bench.json 2> gpurun_out/r2s3m_bench.err; echo "bench rc=$?" >> gpurun_out/r2s3m_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2s3m_ref.json 2> gpurun_out/r2s3m_ref.err; echo "ref rc=$?" >> gpurun_out/r2s3m_ref.err
SKIP_K5=1 timeout 1500 bash tools/profile_bench.sh gpurun_out/r2s3m_prof > gpurun_out/r2s3m_prof.log 2>&1; echo "prof rc=$?" >> gpurun_out/r2s3m_prof.log
