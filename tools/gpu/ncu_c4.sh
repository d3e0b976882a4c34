set -x
mkdir -p gpurun_out
python tests/perf_probe.py C4 > gpurun_out/ncu_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_refine -s 2 -c 1 -o gpurun_out/prof_refine_c4 -f python tests/perf_probe.py C4 > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"
