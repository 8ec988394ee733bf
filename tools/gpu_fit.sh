timeout 600 python -m pytest tests/test_gpu_limits.py tests/test_gpu_fit.py tests/test_gpu_configs.py tests/test_gpu_dexp.py -q -x > gpurun_out/fit.log 2>&1; tail -1 gpurun_out/fit.log
for c in c5 c4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$c', d['ms_per_step'], d['parity']['golden_match'])"; done
