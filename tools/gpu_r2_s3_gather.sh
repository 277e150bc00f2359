# same-box A/B: A = padded tile (before), B = swizzled tile, D = swizzled tile + 8-row x 4-group gather map
# (rt_gather_pos); ncu counters of k_pack_rq_sym for A and D; then the GPU tests touching R (in-tree lib = D)
for rep in 1 2; do for L in A B D; do
  python tools/time_shape.py 17 5 20349 20 --kernels lib=abl/lib$L.so 2>&1 | tail -2 | sed "s#^#c4 lib$L #"
  python tools/time_shape.py 12 6 12376 20 --kernels lib=abl/lib$L.so 2>&1 | tail -2 | sed "s#^#c3 lib$L #"
done; done
for rep in 1 2 3; do for L in A B D; do
  python tools/time_shape.py 10 5 2002 400 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2 lib$L #"
  python tools/time_shape.py 10 5 4004 400 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2b lib$L #"
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
for L in A D; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_pack_rq_sym -s 2 -c 2 --csv python tools/time_shape.py 17 5 20349 4 lib=abl/lib$L.so > gpurun_out/s3_ncu_pack_$L.csv 2>&1
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_oracle_descent.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
