# narrow tiles (diagonal-aligned forward tiles, narrow last column block): GPU tests, then A/B
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/nt_tests.log 2>&1; echo rc=$? >> gpurun_out/nt_tests.log
for v in 0 1 0 1 0 1; do
  SOS_NARROW_TILES=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nt_$v.json 2>/dev/null
  echo "c4 narrow=$v $(python -c "import json;d=json.load(open('gpurun_out/nt_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/nt.log
done
for v in 0 1 0 1; do
  SOS_NARROW_TILES=$v timeout 300 python bench.py --workload c3_n12_2d12 --steps 40 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nt3_$v.json 2>/dev/null
  echo "c3 narrow=$v $(python -c "import json;d=json.load(open('gpurun_out/nt3_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/nt.log
done
