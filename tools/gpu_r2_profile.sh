# round-2 evidence: bench line, ncu launch list (durations + DRAM bytes), ncu --set full of the hot
# kernels at config 4, the fused update measured alone (experiment build, SOS_GEMM_PROBE=8), the
# split step's launch list at config 2, and the config sweep (graph replay timing)
set -x
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/p2_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/p2_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemmq|k_pack_rq_sym|k_rmax_level" -s 4 -c 6 -o gpurun_out/p2_c4_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/p2_ncu2.log 2>&1
python -c "from paper_2410_19844_b200 import build; build.build(experiments=True)"
for shape in "17 5 20349" "12 6 12376"; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_gemmq -c 8 --csv --log-file "gpurun_out/p2_probe8_${shape// /_}.csv" env SOS_GEMM_PROBE=8 python tools/time_shape.py $shape 3 --exp > /dev/null 2>&1
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_gemmq -c 8 --csv --log-file "gpurun_out/p2_probe0_${shape// /_}.csv" python tools/time_shape.py $shape 3 > /dev/null 2>&1
done
timeout 300 ncu --metrics $M --clock-control none -c 80 --csv --log-file gpurun_out/p2_launches_c2.csv python tools/time_shape.py 10 5 2002 6 > /dev/null 2>&1
bash tools/sweep_configs.sh > gpurun_out/p2_sweep.jsonl 2>/dev/null
echo done
