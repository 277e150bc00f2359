# V^T slices: forward aux warps (SOS_VTQ_AUX=1) vs all-SM k_pack_vtq (=0) vs the size rule (-1)
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/vt_tests.log 2>&1; echo rc=$? >> gpurun_out/vt_tests.log
for v in -1 0 1 -1 0 1; do
  echo "vtq_aux=$v" >> gpurun_out/vt.log
  SOS_VTQ_AUX=$v timeout 300 python bench.py --workload c2_n10_2d10 --steps 500 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/vt_c2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vt_c2.json'));k=d['kernels'];print('  c2',round(d['value'],1),round(k['gemm_fwd']['ms_per_launch']*1e3,1),round(k['pack_v']['ms_per_launch']*1e3,1),round(k['gemm_bwd']['ms_per_launch']*1e3,1))" >> gpurun_out/vt.log
  SOS_VTQ_AUX=$v timeout 300 python tools/time_shape.py 100 2 5050 40 >> gpurun_out/vt.log 2>&1
  SOS_VTQ_AUX=$v timeout 300 python bench.py --workload c3_n12_2d12 --steps 60 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vt_c3.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vt_c3.json'));k=d['kernels'];print('  c3',round(d['value'],2),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['pack_v']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))" >> gpurun_out/vt.log
done
for v in -1 0; do
  SOS_VTQ_AUX=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vt_c4.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/vt_c4.json'));k=d['kernels'];print('  c4 vtq_aux=$v',round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))" >> gpurun_out/vt.log
done
