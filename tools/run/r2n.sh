set -u
probe() {
  for c in c3; do python tools/c2_k1_probe.py $c; done
  python bench.py --no-latency --no-e2e --no-cpu-baseline --no-configs --steps 10 --quiet | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('value', round(d['value']), 'K1', round(k['K1_hash']['gbs']), 'K2', round(k['K2_diff']['gbs']), 'fused', round(d['fused_step']['K5_plus_filtered_K2']['gbs']), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
echo "== L2::256B prefetch" > gpurun_out/r2n_ab.txt
probe >> gpurun_out/r2n_ab.txt 2>&1
sed -i 's/#define KC_CP_L2_PREFETCH 1/#define KC_CP_L2_PREFETCH 0/' paper_2605_03208_b200/csrc/kc_kernels.cu
python -c "from paper_2605_03208_b200 import build as b; b.build_lib(force=True)" >> gpurun_out/r2n_build.log 2>&1
echo "== no prefetch hint" >> gpurun_out/r2n_ab.txt
probe >> gpurun_out/r2n_ab.txt 2>&1
sed -i 's/#define KC_CP_L2_PREFETCH 0/#define KC_CP_L2_PREFETCH 1/' paper_2605_03208_b200/csrc/kc_kernels.cu
python -c "from paper_2605_03208_b200 import build as b; b.build_lib(force=True)" >> gpurun_out/r2n_build.log 2>&1
echo "== L2::256B prefetch again" >> gpurun_out/r2n_ab.txt
probe >> gpurun_out/r2n_ab.txt 2>&1
