# R preparation rework (cooperative lattice DP with colex successor, PT prefetch in the packer, one fixup
# launch): full GPU suite, per-kernel times and an ncu launch list at config 4
python -m pytest tests -q -m gpu -x > gpurun_out/r2_tests_b.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2_tests_b.log
for s in "12 6 12376" "17 5 20349"; do timeout 300 python tools/time_shape.py $s 10 --kernels; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c4_b.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-loss-grad > /dev/null 2>&1
python bench.py --no-cpu-baseline > gpurun_out/r2_bench_b.json 2>/dev/null; tail -c 400 gpurun_out/r2_bench_b.json
