# A/B: forward last-wave K split (SOS_FWD_SPLIT) on config 3 (1960 tiles = 26 waves + 36) and config 4
for v in 0 1 0 1 0 1; do
  SOS_FWD_SPLIT=$v timeout 300 python bench.py --workload c3_n12_2d12 --steps 40 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fs3_$v.json 2>/dev/null
  echo "c3 fsplit=$v $(python -c "import json;d=json.load(open('gpurun_out/fs3_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/fs.log
done
for v in 0 1 0 1; do
  SOS_FWD_SPLIT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fs4_$v.json 2>/dev/null
  echo "c4 fsplit=$v $(python -c "import json;d=json.load(open('gpurun_out/fs4_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/fs.log
done
