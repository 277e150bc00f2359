python -m pytest tests -q -m gpu -x -k "variants or oracle_descent or full_size_descend or descend_matches or solve_host or descent_full_size" 2>&1 | tail -3
for s in "12 6 12376" "17 5 20349"; do for h in 0 1; do timeout 300 python tools/time_shape.py $s 10 r_headroom=$h --kernels; done; done
