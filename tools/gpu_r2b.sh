# round-2 profiles: launch lists of C3/C4 and a full capture of the C3 kernels + C4 top-r
mkdir -p gpurun_out
for c in c3 c4; do
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$c.csv \
  python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"nz_encode|crc_chunks|bm_scatter|bm_counts" -c 8 -o gpurun_out/full_c3 -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c3.log 2>&1
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"topr_" -c 10 -o gpurun_out/full_c4topr -f \
  python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c4topr.log 2>&1
tail -2 gpurun_out/full_c3.log gpurun_out/full_c4topr.log
ls -la gpurun_out/
