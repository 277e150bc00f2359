# column-major forward scatter: same-box A/B against the previous build (lib=... A side)
A=paper_2410_19844_b200/libsos_b200_A.so
for s in "8 4 330" "10 5 2002" "10 5 4004" "20 2 210" "76 2 2926" "12 6 12376" "17 5 20349"; do
  for rep in 1 2; do
    timeout 300 python tools/time_shape.py $s 200 lib=$A | sed 's/^/A /'
    timeout 300 python tools/time_shape.py $s 200 | sed 's/^/B /'
  done
done
timeout 120 python tools/time_shape.py 10 5 2002 50 --kernels lib=$A | sed 's/^/A /'
timeout 120 python tools/time_shape.py 10 5 2002 50 --kernels | sed 's/^/B /'
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
