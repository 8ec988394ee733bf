ncu --set full --import-source on --clock-control none --cache-control none -k regex:"topr_" -c 4 -o gpurun_out/full_topr -f \
  python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_topr.log 2>&1
tail -1 gpurun_out/full_topr.log
