# ms/step of several configs: bash tools/gpu_cfgs.sh "c4 c3 c3r"
for c in ${1:-c4}; do
timeout 180 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$c', d['ms_per_step'], d['roofline']['kernel'], d['roofline']['ms_per_launch'])"
done
