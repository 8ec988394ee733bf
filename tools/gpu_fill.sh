timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_fill.log 2>&1; tail -1 gpurun_out/t_fill.log
for f in 1 0; do for c in c4 c1 c2 c3; do
GP_FILL_KERNEL=$f python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/err_$c.log; python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('fill $f $c', d['ms_per_step'], d['value'], d.get('parity',{}).get('golden_match'), d.get('gpu_launches'))"; done; done
