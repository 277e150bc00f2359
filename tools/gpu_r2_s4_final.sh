# fourth-session final evidence at HEAD: smoke, the full GPU suite, the default bench line, the reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f_smoke.log 2>&1; echo smoke_rc=$?
python -m pytest tests -q -m gpu --durations=8 > gpurun_out/s4f_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s4f_tests.log
timeout 900 python bench.py > gpurun_out/s4f_bench.json 2> gpurun_out/s4f_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s4f_reference.json 2> gpurun_out/s4f_reference.err; echo ref_rc=$?
