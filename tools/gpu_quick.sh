# parity suites + C4 bench + C4 launch list
python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python bench.py --config ${1:-c4} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_q.json 2> gpurun_out/err_q.log
python -c "
import json; d=json.load(open('gpurun_out/b_q.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], {k:round(v,3) for k,v in d.get('stages_ms_per_step').items()})"
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/l_q.csv \
  python bench.py --config ${1:-c4} --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
