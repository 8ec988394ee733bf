ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"bloom_members|topr_hist|topr_select|crc_chunks|p2_pairs|p2_scatter|p2_engine|radix_onesweep|fit_segment|members_compact|flags_compact" \
  -c 22 -o gpurun_out/full_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c4.log 2>&1
tail -1 gpurun_out/full_c4.log
ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"nz_encode|crc_chunks|bm_scatter|bm_counts" -c 8 -o gpurun_out/full_c3 -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c3.log 2>&1
tail -1 gpurun_out/full_c3.log
