# K-skew retune with serpentine K + forward split on
run() { tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sk_$tag.json 2>/dev/null
  echo "$tag $* $(python -c "import json;d=json.load(open('gpurun_out/sk_$tag.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],3),round(k['gemm_bwd']['ms_per_launch'],3))")" >> gpurun_out/sk.log
}
for rep in 1 2; do
run a$rep SOS_SKEW_EPOCH=4 SOS_SKEW_LAG=2
run c$rep SOS_SKEW_EPOCH=8 SOS_SKEW_LAG=1
run h$rep SOS_SKEW_EPOCH=12 SOS_SKEW_LAG=1
run i$rep SOS_SKEW_EPOCH=6 SOS_SKEW_LAG=2
run j$rep SOS_SKEW_EPOCH=16 SOS_SKEW_LAG=1
done
