set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_rigs.py tests/test_gpu_parity_c1.py tests/test_gpu_parity_fuzz.py -q -x -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r2d_tests.log
timeout 900 python tools/ab_probe.py C3 "" > gpurun_out/r2d_ab.log 2>&1; tail -1 gpurun_out/r2d_ab.log
