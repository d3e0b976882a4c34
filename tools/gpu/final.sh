# Round-end evidence run: full GPU suite, bench lines for every config, launch list, ncu of k_refine
set -x
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final/gpu.txt
lscpu | head -20 > gpurun_out/final/cpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > gpurun_out/final/pytest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/final/pytest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
echo "bench c3 rc=$?"
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_ref_c3.json 2> gpurun_out/final/bench_ref_c3.err
echo "bench ref rc=$?"
for c in C2 C4 C5 C3G; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
python tests/perf_probe.py C3 > gpurun_out/final/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_refine -s 2 -c 1 -o gpurun_out/final/prof_refine -f \
    python tests/perf_probe.py C3 > gpurun_out/final/ncu_refine.log 2>&1
echo "ncu refine rc=$?"
