# round-2 first check: config-size parity suite, the whole GPU suite, default bench with parity
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_configs.py -q -x > gpurun_out/cfg.log 2>&1; tail -15 gpurun_out/cfg.log
python -m pytest tests -q -m gpu > gpurun_out/t.log 2>&1; tail -8 gpurun_out/t.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; head -c 4000 gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
for c in c3 c4s c1; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/err_$c.log
python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d['parity'])"
tail -3 gpurun_out/err_$c.log
done
