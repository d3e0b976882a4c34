# A/B of grid-rig projection variants on C4 (VARS), ncu of the last one
set -x
mkdir -p gpurun_out
export LFDG_ALLOW_MISSING_SYMBOLS=1
cp paper_1812_06856_b200/liblfdg.so /tmp/liblfdg.main.so
for v in ${VARS}; do
  cp build/variants/$v/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 900 python tools/ab_probe.py C4 "LFDG_VARIANT=$v" >> gpurun_out/${TAG}.log 2>&1
done
if [ -n "$NCUV" ]; then
  cp build/variants/$NCUV/liblfdg.so paper_1812_06856_b200/liblfdg.so
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_refine -s 2 -c 1 -o gpurun_out/prof_${TAG} -f \
      python tests/perf_probe.py C4 > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"
fi
cp /tmp/liblfdg.main.so paper_1812_06856_b200/liblfdg.so
