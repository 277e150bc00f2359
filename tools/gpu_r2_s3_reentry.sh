python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo smoke_rc=$?
python -m pytest tests -q -m gpu --durations=8 > gpurun_out/s3_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/s3_tests.log
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench_rc=$?
