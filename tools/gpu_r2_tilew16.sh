# tile widths that are multiples of 16 (not 32): parity first, then forced widths per shape
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -3
for s in "8 4 330" "10 5 2002" "10 5 4004" "20 2 210" "30 2 465" "76 2 2926"; do
  for w in 0 160 144 128 112 96; do
    timeout 300 python tools/time_shape.py $s 200 tile_w=$w
  done
done
timeout 120 python tools/time_shape.py 10 5 2002 50 --kernels tile_w=128
timeout 120 python tools/time_shape.py 10 5 2002 50 --kernels tile_w=112
