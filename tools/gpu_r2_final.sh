# round-2 final evidence on the final build: full GPU suite, smoke, default bench line (config 4, with cpu_baseline),
# config sweep, split-step ncu (config 2) launch list + --set full, config-4 launch list, paper table
set -x
python -m pytest tests -q -m gpu --durations=8 > gpurun_out/f_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench_rc=$?
bash tools/sweep_configs.sh > gpurun_out/f_sweep.jsonl 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none -c 60 --csv --log-file gpurun_out/f_launches_c2_split.csv python tools/time_shape.py 10 5 2002 6 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update_rows|k_mid|k_gemmq" -s 8 -c 4 -o gpurun_out/f_split_c2 python tools/time_shape.py 10 5 2002 6 > gpurun_out/f_ncu_split.log 2>&1
timeout 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/f_ncu_c4.log 2>&1
timeout 900 python tools/paper_table.py --out gpurun_out/f_paper_table.md > gpurun_out/f_paper_table.log 2>&1
echo done
