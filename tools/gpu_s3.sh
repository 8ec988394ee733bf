# session-3 check: GPU suite at HEAD + C3/C4 bench lines
python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for c in ${@:-c3 c4}; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/err_$c.log
python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d.get('parity'), {k:round(v,3) for k,v in d.get('stages_ms_per_step').items()})"
done
