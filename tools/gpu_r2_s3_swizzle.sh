# same-box A/B of the swizzled R tile (rt_slot) in the R packers: A = HEAD before, B = swizzled,
# C = swizzled with __launch_bounds__(256, 5) on k_pack_rq_sym (no spill); then the GPU tests touching R
for rep in 1 2; do for L in A B C; do
  python tools/time_shape.py 17 5 20349 20 --kernels lib=abl/lib$L.so 2>&1 | tail -2 | sed "s#^#c4 lib$L #"
done; done
for rep in 1 2; do for L in A B C; do
  python tools/time_shape.py 12 6 12376 20 --kernels lib=abl/lib$L.so 2>&1 | tail -2 | sed "s#^#c3 lib$L #"
done; done
for rep in 1 2 3; do for L in A B; do
  python tools/time_shape.py 10 5 2002 400 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2 lib$L #"
  python tools/time_shape.py 10 5 2002 400 split=1 rmax_direct=1 lib=abl/lib$L.so 2>&1 | tail -1 | sed "s#^#c2 lib$L #"
done; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_oracle_descent.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
