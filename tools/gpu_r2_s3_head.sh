# third-session final evidence on HEAD: full GPU suite, smoke, default bench line, config sweep, config-4 launch list
python -m pytest tests -q -m gpu --durations=5 > gpurun_out/s3h_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s3h_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3h_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/s3h_bench.json 2> gpurun_out/s3h_bench.err; echo bench_rc=$?
bash tools/sweep_configs.sh > gpurun_out/s3h_sweep.jsonl 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/s3h_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/s3h_ncu_c4.log 2>&1
timeout 300 ncu --metrics $M --clock-control none -c 60 --csv --log-file gpurun_out/s3h_launches_c2_split.csv python tools/time_shape.py 10 5 2002 6 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pack_rq_sym" -s 2 -c 1 -o gpurun_out/s3h_pack_full python tools/time_shape.py 17 5 20349 4 > gpurun_out/s3h_ncu_pack_full.log 2>&1
echo done
