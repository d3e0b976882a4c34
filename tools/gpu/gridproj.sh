# A/B of the grid-rig projection mode (kFlat 4) on C4, then the parity tests that cover it
set -x
mkdir -p gpurun_out
export LFDG_ALLOW_MISSING_SYMBOLS=1
cp paper_1812_06856_b200/liblfdg.so /tmp/liblfdg.main.so
for v in gp0 gp1; do
  cp build/variants/$v/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 900 python tools/ab_probe.py C4 "LFDG_VARIANT=$v" >> gpurun_out/gp.log 2>&1
done
cp /tmp/liblfdg.main.so paper_1812_06856_b200/liblfdg.so
timeout 1200 python -m pytest tests/test_gpu_parity_rigs.py tests/test_gpu_parity_configs.py tests/test_gpu_parity_fuzz.py -q -x -p no:cacheprovider > gpurun_out/gp_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gp_tests.log
