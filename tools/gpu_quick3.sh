# quick check: dense-path tests + config parity + C3/C4 bench lines
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dense.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for c in ${CONFIGS:-c3 c4}; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_$c.json 2> gpurun_out/q_err_$c.log
python -c "
import json; d=json.load(open('gpurun_out/q_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d['parity']['golden_match'], d.get('stages_ms_per_step'))"
tail -2 gpurun_out/q_err_$c.log
done
