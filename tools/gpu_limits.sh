mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_limits.py -q -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_dexp.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -4
CONFIGS="c4 c1" bash tools/gpu_quick3.sh 2>&1 | grep -v passed | tail -3
