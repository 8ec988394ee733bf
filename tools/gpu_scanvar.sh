python -m pytest tests -q -m gpu -x -k "bloom or P1 or P2 or naive or pd or p0 or Bloom" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in ${VARS:-0 1 2 3 4 5}; do for c in ${CFGS:-c4 c1}; do
GP_SCAN_VARIANT=$v python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_s.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_s.json')); st=d['stages_ms_per_step']; print('v$v $c', d['ms_per_step'], st['bloom_scan'], st['dec_bloom_scan'])"
done; done
