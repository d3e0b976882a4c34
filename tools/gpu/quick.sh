# quick correctness + C3 timing of the current build (dev loop)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_c1.py tests/test_gpu_parity_rigs.py tests/test_gpu_parity_c2_full.py -q -x -p no:cacheprovider > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/quick_tests.log
timeout 600 python tests/perf_probe.py C3 > gpurun_out/quick_probe.log 2>&1
echo "probe rc=$?"; tail -3 gpurun_out/quick_probe.log
