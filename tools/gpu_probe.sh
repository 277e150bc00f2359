# experiment: power share of the operand memory system (SOS_GEMM_PROBE, wrong results by design)
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pr_$tag.json 2> gpurun_out/pr_$tag.err
  echo "$tag $* $(python -c "import json;d=json.load(open('gpurun_out/pr_$tag.json'));k=d['kernels'];print(round(d['value'],3),d['clocks']['sm_mhz'],round(k['gemm_fwd']['ms_per_launch'],2),round(k['gemm_bwd']['ms_per_launch'],2))")" >> gpurun_out/pr2.log
}
run b SOS_GEMM_PROBE=2
run c SOS_GEMM_PROBE=4
run d SOS_GEMM_PROBE=2
run e SOS_GEMM_PROBE=4
