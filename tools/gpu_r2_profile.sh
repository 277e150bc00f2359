# round-2 evidence: bench line, ncu launch list (durations + DRAM bytes), ncu --set full of the hot
# kernels at config 4, the split step's launch list at config 2, and the config sweep (graph
# replay timing)
set -x
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/p2_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/p2_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemmq|k_pack_rq_sym|k_rmax_level" -s 4 -c 6 -o gpurun_out/p2_c4_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/p2_ncu2.log 2>&1
timeout 300 ncu --metrics $M --clock-control none -c 80 --csv --log-file gpurun_out/p2_launches_c2.csv python tools/time_shape.py 10 5 2002 6 > /dev/null 2>&1
bash tools/sweep_configs.sh > gpurun_out/p2_sweep.jsonl 2>/dev/null
echo done
