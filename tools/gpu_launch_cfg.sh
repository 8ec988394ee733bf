# usage: CFG=c4ef bash tools/gpu_launch_cfg.sh
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$CFG.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
