mkdir -p gpurun_out/cfg
for c in c4 c4s c4ef c3 c3r c1 c2 c2r c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg/bench_$c.json 2> gpurun_out/cfg/err_$c.log
  python -c "
import json; d=json.load(open('gpurun_out/cfg/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d.get('bits_per_nonzero'), (d.get('parity') or {}).get('golden_match'), d.get('cpu_baseline',{}).get('seconds'))" || tail -3 gpurun_out/cfg/err_$c.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/cfg/bench_c4_reference.json 2> gpurun_out/cfg/err_ref.log; head -c 600 gpurun_out/cfg/bench_c4_reference.json
