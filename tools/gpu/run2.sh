set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_parity_rigs.py tests/test_gpu_pipelined_transfers.py tests/test_gpu_bench_contract.py -q -x -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2b_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c3.json 2> gpurun_out/r2b_bench_c3.err
echo "bench rc=$?"
timeout 900 python bench.py --config C3G --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_c3g.json 2> gpurun_out/r2b_bench_c3g.err
echo "bench c3g rc=$?"
timeout 1500 python tools/validate_cpu_extrapolation.py C1 C2 > gpurun_out/r2b_cpu_validate.log 2>&1
echo "validate rc=$?"; cat gpurun_out/r2b_cpu_validate.log | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_slic_assign|k_slic_update|k_rasterize|k_build_raster' -s 40 -c 4 -o gpurun_out/prof_slic_rast -f python tests/perf_probe.py C3 > gpurun_out/r2b_ncu.log 2>&1
echo "ncu rc=$?"
