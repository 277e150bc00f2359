# column tile width A/B (same box): 160 vs 128 vs auto
for s in "8 4 330" "10 5 2002" "10 5 4004" "20 2 210" "30 2 465" "76 2 2926"; do
  for w in 160 128 0; do timeout 300 python tools/time_shape.py $s 400 tile_w=$w; done
done
