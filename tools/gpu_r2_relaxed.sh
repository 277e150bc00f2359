python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for s in "8 4 330" "10 5 2002" "10 5 4004" "20 2 210" "30 2 465" "76 2 2926" "12 6 12376" "17 5 20349"; do timeout 300 python tools/time_shape.py $s 100; done
SOS_GEMM_TRACE=1 timeout 120 python tools/time_shape.py 8 4 330 2 --exp 2>&1 | grep -E "cta0 \(us\)" | tail -2
