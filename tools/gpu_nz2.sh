for m in 1 0; do
GP_NZ_MODE=$m python -m pytest tests/test_gpu_dense.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -k "c3 or dense or bitmap or Dense or nz" > gpurun_out/t_nz$m.log 2>&1; echo "mode $m: $(tail -1 gpurun_out/t_nz$m.log)"
done
for m in 1 7 8 0; do
GP_NZ_MODE=$m python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_nz$m.json 2> gpurun_out/err_nz$m.log
python -c "
import json; d=json.load(open('gpurun_out/b_nz$m.json')); print('mode $m', d['ms_per_step'], d.get('parity',{}).get('golden_match'), {k:round(v,4) for k,v in d.get('stages_ms_per_step').items()})"
done
