# A/B timing (tools/ab_probe.py) + quick parity
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_c1.py tests/test_gpu_parity_rigs.py tests/test_gpu_parity_c2_full.py -q -x -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
timeout 900 python tools/ab_probe.py ${CFG:-C3} ${VARIANTS} > gpurun_out/ab_${TAG:-x}.log 2>&1
echo "ab rc=$?"; cat gpurun_out/ab_${TAG:-x}.log | tail -6
