# usage: bash tools/ncu_kernel.sh <config> <kernel-regex> <out-name> [count]
cfg=$1; kr=$2; out=$3; cnt=${4:-1}
ncu --set full --import-source on --clock-control none --cache-control none -k regex:$kr -c $cnt -o gpurun_out/$out -f \
  python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$out.log 2>&1
tail -2 gpurun_out/$out.log
