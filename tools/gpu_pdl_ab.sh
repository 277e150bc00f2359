# programmatic dependent launch (SOS_PDL=1, default) vs plain stream order (=0)
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pdl_tests.log 2>&1; echo rc=$? >> gpurun_out/pdl_tests.log
for v in 1 0 1 0; do
  for w in c1_n8_2d8:2000 c2_n10_2d10:1000 c2b_n10_2d10_r4004:600 c3_n12_2d12:60 c4_n17_2d10:20; do
    SOS_PDL=$v timeout 300 python bench.py --workload ${w%%:*} --steps ${w##*:} --warmup 5 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/pdl.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/pdl.json'));print('pdl=$v ${w%%:*}',round(d['value'],2),round(d['ms_per_step'],4))" >> gpurun_out/pdl.log
  done
done
