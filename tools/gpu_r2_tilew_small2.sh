timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -3
for s in "8 4 330" "20 2 210" "30 2 465" "9 4 495" "11 4 1001" "10 5 2002" "8 4 4000" "10 5 600"; do
  for w in 0 64 32 16; do
    timeout 300 python tools/time_shape.py $s 200 tile_w=$w
  done
done
timeout 120 python tools/time_shape.py 8 4 330 50 --kernels
