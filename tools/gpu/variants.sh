# Time each prebuilt library variant under build/variants/<name>/liblfdg.so with tools/ab_probe.py
set -x
mkdir -p gpurun_out
cp paper_1812_06856_b200/liblfdg.so /tmp/liblfdg.main.so
for v in ${VARS}; do
  cp build/variants/$v/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 600 python tools/ab_probe.py ${CFG:-C3} "LFDG_VARIANT=$v" >> gpurun_out/var_${TAG:-x}.log 2>&1
done
cp /tmp/liblfdg.main.so paper_1812_06856_b200/liblfdg.so
cat gpurun_out/var_${TAG:-x}.log
