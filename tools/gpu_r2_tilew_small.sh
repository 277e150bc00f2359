# widths below 96 on one-wave problems (forced; tile_w=0 = auto)
for s in "8 4 330" "20 2 210" "30 2 465" "9 4 495" "11 4 1001" "10 5 2002"; do
  for w in 0 96 80 64 48 32; do
    timeout 300 python tools/time_shape.py $s 200 tile_w=$w
  done
done
timeout 120 python tools/time_shape.py 8 4 330 50 --kernels tile_w=48
