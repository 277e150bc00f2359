# grouped-raster height (SOS_TILE_GROUP) with the current build, interleaved repeats
for rep in 1 2 3; do for ga in 8 6 10 12 16; do
  SOS_TILE_GROUP=$ga timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ga.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ga.json'));k=d['kernels'];print('ga=$ga',round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))" >> gpurun_out/ga.log
done; done
