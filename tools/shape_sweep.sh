python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "bloom or P1 or P2 or naive or pd or p0" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for sh in 44 48 84 88 162; do
GP_BLOOM_SHAPE=$sh python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_s.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_s.json')); st=d['stages_ms_per_step']; print('$sh', d['ms_per_step'], st['bloom_scan'], st['dec_bloom_scan'])"
done
