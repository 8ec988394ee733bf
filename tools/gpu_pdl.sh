timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_pdl.log 2>&1; tail -2 gpurun_out/t_pdl.log
for p in 1 0; do for c in c2 c1 c4 c3; do
GP_PDL=$p python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/err_$c.log; python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('pdl $p $c', d['ms_per_step'], d['value'], d.get('parity',{}).get('golden_match'))"; done; done
