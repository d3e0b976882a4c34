set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -q -x -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2c_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2c_bench_c3.json 2> gpurun_out/r2c_bench_c3.err
echo "bench rc=$?"
timeout 900 python bench.py --config C3G --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_c3g.json 2> gpurun_out/r2c_bench_c3g.err
echo "bench c3g rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_rasterize|k_build_raster|k_sweep' -s 3 -c 3 -o gpurun_out/prof_rast_sweep -f python tests/perf_probe.py C3 > gpurun_out/r2c_ncu.log 2>&1
echo "ncu rc=$?"
