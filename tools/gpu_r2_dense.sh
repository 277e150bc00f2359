python -m pytest tests -q -m gpu -x -k "forward_parity or fuzz or boundary or config1 or config0 or tiny or smoke" 2>&1 | tail -2
for s in "8 4 330" "20 2 210" "25 2 325" "30 2 465" "10 5 2002" "5 3 35"; do timeout 300 python tools/time_shape.py $s 400; done
SOS_GEMM_TRACE=1 timeout 120 python tools/time_shape.py 8 4 330 2 --exp 2>&1 | grep -E "k_gemmq<0> cta0 \(us\)" | tail -1
