set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x --durations=25 -p no:cacheprovider > gpurun_out/pytest_r2a.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2a.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_r2a.json
