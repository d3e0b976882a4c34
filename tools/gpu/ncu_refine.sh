# ncu --set full of one k_refine launch (C3, l = 3) + the plain run before it
set -x
mkdir -p gpurun_out
python tests/perf_probe.py C3 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_refine -s 2 -c 1 -o gpurun_out/prof_refine_${TAG:-x} -f \
    python tests/perf_probe.py C3 > gpurun_out/ncu_refine_${TAG:-x}.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_refine_${TAG:-x}.log
