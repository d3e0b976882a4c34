set -x
mkdir -p gpurun_out
python tests/perf_probe.py C3 > gpurun_out/ncu_plain_sw.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/prof_sweep_${TAG:-x} -f \
    python tests/perf_probe.py C3 > gpurun_out/ncu_sweep_${TAG:-x}.log 2>&1
echo "ncu rc=$?"
