timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_limits.py -q -x -k "bloom or config or p2" > gpurun_out/p2_tests.log 2>&1; tail -1 gpurun_out/p2_tests.log
timeout 300 bash tools/gpu_launch_c4.sh
