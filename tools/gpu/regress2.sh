set -x
mkdir -p gpurun_out
export LFDG_ALLOW_MISSING_SYMBOLS=1
cp paper_1812_06856_b200/liblfdg.so /tmp/liblfdg.main.so
for cfg in ${CFGS:-C3 C5 C4}; do
for v in ${VARS}; do
  cp build/variants/$v/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 900 python tools/ab_probe.py $cfg "LFDG_VARIANT=$v,CFG=$cfg" >> gpurun_out/${TAG:-regress2}.log 2>&1
done
done
cp /tmp/liblfdg.main.so paper_1812_06856_b200/liblfdg.so
timeout 900 python -m pytest tests/test_gpu_parity_c1.py tests/test_gpu_parity_rigs.py tests/test_gpu_parity_c2_full.py tests/test_gpu_parity_fuzz.py -q -x -p no:cacheprovider > gpurun_out/${TAG:-regress2}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${TAG:-regress2}_tests.log
