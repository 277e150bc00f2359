# split update (gradient via HBM + all-SM k_update) vs the fused epilogue update, by K length
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/us_tests.log 2>&1; echo rc=$? >> gpurun_out/us_tests.log
for v in 0 1 0 1; do
  echo "update_split=$v" >> gpurun_out/us.log
  for w in c1_n8_2d8:2000 c2_n10_2d10:1000 c2b_n10_2d10_r4004:600; do
    SOS_UPDATE_SPLIT=$v timeout 300 python bench.py --workload ${w%%:*} --steps ${w##*:} --warmup 5 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/us.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/us.json'));k=d['kernels'];print('  ${w%%:*}',round(d['value'],1),round(k['gemm_bwd']['ms_per_launch']*1e3,1),round(k['update']['ms_per_launch']*1e3,1))" >> gpurun_out/us.log
  done
  SOS_UPDATE_SPLIT=$v timeout 300 python tools/time_shape.py 100 2 5050 40 >> gpurun_out/us.log 2>&1
  SOS_UPDATE_SPLIT=$v timeout 300 python tools/time_shape.py 20 3 3000 100 >> gpurun_out/us.log 2>&1
done
