mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ef64.py -q -x 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
