# time prebuilt library variants (build/variants/<name>) with tools/ab_probe.py on ${CFG}; optional ncu of ${NCUK} on ${NCUV}
set -x
mkdir -p gpurun_out
cp paper_1812_06856_b200/liblfdg.so /tmp/liblfdg.main.so
for v in ${VARS}; do
  cp build/variants/$v/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 900 python tools/ab_probe.py ${CFG:-C3} "LFDG_VARIANT=$v" >> gpurun_out/px_var_${TAG:-x}.log 2>&1
done
if [ -n "$NCUK" ]; then
  cp build/variants/${NCUV}/liblfdg.so paper_1812_06856_b200/liblfdg.so
  ncu --set full --clock-control none --import-source on -k regex:$NCUK -s 2 -c 1 -o gpurun_out/prof_${NCUV} -f python tests/perf_probe.py ${CFG:-C3} > gpurun_out/ncu_${NCUV}.log 2>&1
  echo "ncu rc=$?"
fi
cp /tmp/liblfdg.main.so paper_1812_06856_b200/liblfdg.so
cat gpurun_out/px_var_${TAG:-x}.log
