# A/B: forward last-wave K split (SOS_FWD_SPLIT) + parity tests of the forward paths
timeout 900 python -m pytest tests -x -q -m gpu -k "forward or descend or full_size or boundary or loss" > gpurun_out/split_tests.log 2>&1; echo rc=$? >> gpurun_out/split_tests.log
for v in 0 1 0 1; do
  SOS_FWD_SPLIT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/split_$v.json 2>/dev/null
  echo "split=$v $(python -c "import json;d=json.load(open('gpurun_out/split_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/split.log
done
