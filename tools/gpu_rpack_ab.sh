for c in c3_n12_2d12 c4_n17_2d10; do
  SOS_RPACK_SYM=0 timeout 300 python tools/rpack_ab.py $c /tmp/g0.npy && SOS_RPACK_SYM=1 timeout 300 python tools/rpack_ab.py $c /tmp/g1.npy && python -c "
import numpy as np; a=np.load('/tmp/g0.npy'); b=np.load('/tmp/g1.npy'); print('$c', 'bit-identical' if np.array_equal(a,b) else 'DIFFER', a.shape)" >> gpurun_out/rp.log
done
for v in 0 1 0 1; do
  SOS_RPACK_SYM=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rp_$v.json 2>/dev/null
  echo "sym=$v $(python -c "import json;d=json.load(open('gpurun_out/rp_$v.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['pack_r']['ms_per_launch'],3),round(k['rmax']['ms_per_launch'],3))")" >> gpurun_out/rp.log
done
timeout 600 python -m pytest tests -x -q -m gpu -k "backward or descend or loss_grad or step" > gpurun_out/rp_tests.log 2>&1; echo rc=$? >> gpurun_out/rp_tests.log
