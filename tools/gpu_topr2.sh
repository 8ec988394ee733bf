timeout 240 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_ef.py tests/test_gpu_dense.py -q -x > gpurun_out/topr_tests.log 2>&1; tail -2 gpurun_out/topr_tests.log
timeout 300 bash tools/gpu_launch_c4.sh
