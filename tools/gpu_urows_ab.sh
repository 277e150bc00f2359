# A/B of the update loop's rows in flight (compile-time SOS_UROWS), small / mid / large shapes
for u in 2 4 8 2 4 8; do
  SOS_NVCC_EXTRA=-DSOS_UROWS=$u python -c "from paper_2410_19844_b200 import build; build.build(force=True)"
  echo "urows=$u" >> gpurun_out/ur.log
  timeout 300 python bench.py --workload c2_n10_2d10 --steps 500 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ur_c2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ur_c2.json'));k=d['kernels'];print('  c2',round(d['value'],1),round(k['gemm_fwd']['ms_per_launch']*1e3,1),round(k['gemm_bwd']['ms_per_launch']*1e3,1))" >> gpurun_out/ur.log
  timeout 300 python tools/time_shape.py 100 2 5050 40 >> gpurun_out/ur.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ur_c4.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ur_c4.json'));k=d['kernels'];print('  c4',round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))" >> gpurun_out/ur.log
done
python -c "from paper_2410_19844_b200 import build; build.build(force=True)"
