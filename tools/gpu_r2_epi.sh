# epilogue column scales in shared memory + PT prefetch: tests, GEMM phase trace, step times
python -m pytest tests -q -m gpu -x -k "parity and not large_n and not descent_full and not config2_adam" 2>&1 | tail -2
for s in "8 4 330" "10 5 2002"; do SOS_GEMM_TRACE=1 timeout 120 python tools/time_shape.py $s 2 --exp 2>&1 | grep -E "k_gemmq" | tail -2; done
for s in "8 4 330" "10 5 2002" "10 5 4004" "12 6 12376" "17 5 20349"; do timeout 300 python tools/time_shape.py $s 20; done
