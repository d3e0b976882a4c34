set -x
mkdir -p gpurun_out
export LFDG_ALLOW_MISSING_SYMBOLS=1
cp paper_1812_06856_b200/liblfdg.so /tmp/liblfdg.main.so
for cfg in C5 C4; do
for v in r1 base1 skip1; do
  cp build/variants/$v/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 900 python tools/ab_probe.py $cfg "LFDG_VARIANT=$v,CFG=$cfg" >> gpurun_out/regress.log 2>&1
done
done
cp /tmp/liblfdg.main.so paper_1812_06856_b200/liblfdg.so
cat gpurun_out/regress.log
