timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_ef.py tests/test_gpu_dense.py -q -x 2>&1 | tail -5
python tools/time_encode.py c4 20
CONFIGS="c4 c3" bash tools/gpu_quick3.sh 2>&1 | grep "^c"
