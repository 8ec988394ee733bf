timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
CONFIGS="c4 c3 c1 c4s" timeout 600 bash tools/gpu_quick3.sh 2>&1 | grep "^c"
