# full round check: GPU parity suites, default bench (with cpu baseline), smoke, launch list
set -x
python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json | head -c 3000; tail -3 gpurun_out/bench_default.err
for c in c1 c2 c3 c5; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/err_$c.log
python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], {k:round(v,3) for k,v in d.get('stages_ms_per_step',{}).items()})"
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; head -c 1500 gpurun_out/bench_ref.json
bash tools/launches.sh c4 launches_c4
