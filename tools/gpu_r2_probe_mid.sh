# cooperative-launch / grid-barrier costs and k_mid phase times (experiment build)
./tools/coop_bench 2>&1 | tee gpurun_out/r2_coop_bench.log
SOS_MID_TRACE=1 python tools/time_shape.py 10 5 2002 3 split=1 --exp 2>&1 | tail -8 | tee gpurun_out/r2_mid_trace_c2.log
SOS_MID_TRACE=1 python tools/time_shape.py 8 4 330 3 split=1 --exp 2>&1 | tail -4 | tee gpurun_out/r2_mid_trace_c1.log
