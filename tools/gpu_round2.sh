# end-of-round evidence: full GPU suite, smoke, default bench + reference arm, all configs, launch list
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; head -c 300 gpurun_out/bench_default.json; echo
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; head -c 200 gpurun_out/bench_ref.json; echo
for c in c1 c2 c3 c3r c2r c4s c4ef c5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/err_$c.log
python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d['bits_per_nonzero'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"bloom_members|members_compact|topr_candidates|topr_hist|p2_scatter|p2_pairs|p2_engine|crc_chunks|radix_onesweep|fit_segment" \
  -c 14 -o gpurun_out/full_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-early > gpurun_out/full_c4.log 2>&1
for c in c3 c1 c5; do
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$c.csv \
  python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
echo profiles-done
