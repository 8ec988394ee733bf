timeout 900 python -m pytest tests/test_gpu_deflate_encode.py -q -x 2>&1 | tail -25
(cd oracle/_ref && timeout 1200 ./acceptance_b200 2>&1 | tail -12)
