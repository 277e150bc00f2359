# next-step V^T slices written by the backward's update (SOS_VTQ_UPDATE=1) vs packed by the forward (=0)
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/vn_tests.log 2>&1; echo rc=$? >> gpurun_out/vn_tests.log
for v in 0 1 0 1; do
  echo "vtq_update=$v" >> gpurun_out/vn.log
  SOS_VTQ_UPDATE=$v timeout 300 python bench.py --workload c2_n10_2d10 --steps 1000 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/vn_c2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vn_c2.json'));k=d['kernels'];print('  c2',round(d['value'],1),round(k['gemm_fwd']['ms_per_launch']*1e3,1),round(k['gemm_bwd']['ms_per_launch']*1e3,1))" >> gpurun_out/vn.log
  SOS_VTQ_UPDATE=$v timeout 300 python tools/time_shape.py 100 2 5050 40 >> gpurun_out/vn.log 2>&1
  SOS_VTQ_UPDATE=$v timeout 300 python bench.py --workload c3_n12_2d12 --steps 60 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vn_c3.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vn_c3.json'));k=d['kernels'];print('  c3',round(d['value'],2),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))" >> gpurun_out/vn.log
  SOS_VTQ_UPDATE=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vn_c4.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vn_c4.json'));k=d['kernels'];print('  c4',round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))" >> gpurun_out/vn.log
done
