# third-session evidence: same-box A/B of the R-tile variants (B = swizzled tile, D = + rt_gather_pos in every
# packer, E = rt_gather_pos in k_pack_rq_sym / k_rmax only, k_mid row-major = the in-tree build), then the full
# GPU suite, smoke, the default bench line, the config sweep and a config-4 launch list on the in-tree build
for rep in 1 2 3; do for L in B D E; do
  python tools/time_shape.py 10 5 2002 400 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2 lib$L #"
  python tools/time_shape.py 10 5 4004 400 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2b lib$L #"
  python tools/time_shape.py 8 4 330 800 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c1 lib$L #"
done; done
for L in B E; do
  python tools/time_shape.py 17 5 20349 20 --kernels lib=abl/lib$L.so 2>&1 | tail -2 | sed "s#^#c4 lib$L #"
done
python -m pytest tests -q -m gpu --durations=5 > gpurun_out/s3f_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s3f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3f_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/s3f_bench.json 2> gpurun_out/s3f_bench.err; echo bench_rc=$?
bash tools/sweep_configs.sh > gpurun_out/s3f_sweep.jsonl 2>/dev/null
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/s3f_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-loss-grad > gpurun_out/s3f_ncu_c4.log 2>&1
M2=$M,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M2 --clock-control none -k regex:k_pack_rq_sym -s 2 -c 2 --csv python tools/time_shape.py 17 5 20349 4 > gpurun_out/s3f_ncu_pack.csv 2>&1
echo done
