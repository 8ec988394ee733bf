# round-2 final evidence at HEAD: GPU suite, smoke, every config's bench line,
# the reference arm, launch lists and ncu full captures (outputs: gpurun_out/final/)
o=gpurun_out/final; mkdir -p $o/cfg
timeout 900 python -m pytest tests -m gpu -q > $o/gpu_suite.txt 2>&1; tail -1 $o/gpu_suite.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/smoke.txt 2>&1; tail -1 $o/smoke.txt
for c in c4 c4s c4ef c3 c3r c1 c2 c2r c5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 > $o/cfg/bench_$c.json 2> $o/cfg/err_$c.log
  python -c "
import json; d=json.load(open('$o/cfg/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d.get('bits_per_nonzero'), (d.get('parity') or {}).get('golden_match'), d.get('gpu_launches'))" || tail -3 $o/cfg/err_$c.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $o/cfg/bench_c4_reference.json 2> $o/cfg/err_ref.log; head -c 300 $o/cfg/bench_c4_reference.json; echo
for c in c4 c3 c1 c2 c4s c5; do
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $o/launches_$c.csv \
  python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"bloom_members|topr_hist|topr_select|crc_tail|p2_pairs|p2_scatter|p2_engine|radix_onesweep|fit_segment|members_compact|flags_compact" \
  -c 22 -o $o/full_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > $o/full_c4.log 2>&1
tail -1 $o/full_c4.log
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"nz_count|nz_write|crc_chunks|bm_scatter|bm_counts" -c 8 -o $o/full_c3 -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > $o/full_c3.log 2>&1
tail -1 $o/full_c3.log
for st in 12 16; do
  timeout 300 python bench.py --config c5 --streams $st --steps 10 --warmup 3 --no-cpu-baseline > $o/c5_streams_$st.json 2>/dev/null
  python -c "import json; d=json.load(open('$o/c5_streams_$st.json')); print('c5 streams $st', d['ms_per_step'])"
done
