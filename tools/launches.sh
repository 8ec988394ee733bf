# usage: bash tools/launches.sh <config> <out-name>
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/$2.csv \
  python bench.py --config $1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
