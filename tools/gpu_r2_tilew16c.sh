A=paper_2410_19844_b200/libsos_b200_A.so
for s in "8 4 330" "10 5 2002" "10 5 4004" "20 2 210" "30 2 465" "76 2 2926" "11 4 1001" "9 4 495" "12 5 4368"; do
  for rep in 1 2; do
    timeout 300 python tools/time_shape.py $s 200 lib=$A | sed 's/^/A /'
    timeout 300 python tools/time_shape.py $s 200 | sed 's/^/B /'
  done
done
timeout 120 python tools/time_shape.py 8 4 330 50 --kernels | sed 's/^/B /'
timeout 120 python tools/time_shape.py 10 5 2002 50 --kernels | sed 's/^/B /'
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5
