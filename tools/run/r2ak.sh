set -u
for i in 1 2; do
  timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2ak_pytest_$i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ak_pytest_$i.log
done
