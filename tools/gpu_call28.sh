timeout 900 python -m pytest tests -x -q -m gpu -k "not descent_full" > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
timeout 600 python tools/paper_table.py > gpurun_out/paper_table2.log 2>&1
