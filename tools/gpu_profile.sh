# round-1 evidence: default bench line, launch list, full ncu of the two GEMMs and the R packer, smoke, full GPU tests
timeout 600 python bench.py > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -c 400 --csv --log-file gpurun_out/prof_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemmq|k_pack_rq_sym|k_rmax_level" -s 4 -c 6 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_ncu2.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof_smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/prof_tests.log 2>&1; echo rc=$? >> gpurun_out/prof_tests.log
