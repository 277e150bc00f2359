# backward last-wave K split: full GPU tests, then A/B (SOS_BWD_SPLIT) on config 4 and config 2
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/bs_tests.log 2>&1; echo rc=$? >> gpurun_out/bs_tests.log
for v in 0 1 0 1; do
  SOS_BWD_SPLIT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bs_$v.json 2>/dev/null
  echo "c4 bsplit=$v $(python -c "import json;d=json.load(open('gpurun_out/bs_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/bs.log
done
for v in 0 1 0 1; do
  SOS_BWD_SPLIT=$v timeout 300 python bench.py --workload c2_n10_2d10 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bs2_$v.json 2>/dev/null
  echo "c2 bsplit=$v $(python -c "import json;d=json.load(open('gpurun_out/bs2_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],4),round(k['gemm_bwd']['ms_per_launch'],4))")" >> gpurun_out/bs.log
done
