set -u
m() { for i in 1 2; do python tools/c2_k1_probe.py c2; python tools/c5_probe.py 65536 1000 | cut -d' ' -f1-6; done; }
echo "== 3-level (IMAD.WIDE || IMADs -> IADD)" > gpurun_out/r2x_ab.txt; m >> gpurun_out/r2x_ab.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_hash.py -m gpu -q -p no:cacheprovider >> gpurun_out/r2x_ab.txt 2>&1
cp tools/run/kc_kernels_prev.cu.txt paper_2605_03208_b200/csrc/kc_kernels.cu
python -c "from paper_2605_03208_b200 import build as b; b.build_lib(force=True)" > /dev/null 2>&1
echo "== committed (SHF->IMAD->IMAD->IMAD.WIDE)" >> gpurun_out/r2x_ab.txt; m >> gpurun_out/r2x_ab.txt 2>&1
