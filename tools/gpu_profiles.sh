# round profiles: launch lists (c4, c3, c1) + one full capture of the C4 top kernels
for c in c4 c3 c1; do
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$c.csv \
  python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"bloom_members|members_compact|topr_candidates|topr_hist|p2_scatter|p2_pairs|p2_engine|crc_chunks|radix_onesweep|fit_segment" \
  -c 14 -o gpurun_out/full_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c4.log 2>&1
tail -2 gpurun_out/full_c4.log
ls -la gpurun_out/
