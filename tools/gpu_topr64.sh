timeout 500 python -m pytest tests/test_gpu_ef64.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_rle.py -q -x > gpurun_out/t64.log 2>&1; tail -2 gpurun_out/t64.log
for c in c4ef c3r; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$c', d['ms_per_step'], d['stages_ms_per_step'].get('topr'))"; done
