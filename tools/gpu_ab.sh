# A/B of an env knob: bash tools/gpu_ab.sh VAR "v1 v2" "c4 c1"
var=$1; vals=$2; cfgs=${3:-c4}
for v in $vals; do for c in $cfgs; do
env $var=$v timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$var=$v $c', d['ms_per_step'], d['value'])"
done; done
