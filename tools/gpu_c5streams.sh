for st in 3 4 6 8 16; do
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --streams $st > gpurun_out/b_s.json 2>gpurun_out/err_s.log
python -c "
import json; d=json.load(open('gpurun_out/b_s.json')); print('streams $st', d['ms_per_step'], d['value'], d['e2e']['value'])"
done
