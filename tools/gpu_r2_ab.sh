# quick GPU check of a change: GPU suite minus the two slowest tests, then the short-K shapes
# (time_shape --kernels) and config 4 per kernel, A/B against lib=$1; k_mid phase trace
python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_parity.py::test_forward_full_vector_config3 --deselect tests/test_gpu_parity.py::test_large_n_sampled > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/ab_tests.log
for s in "8 4 330" "10 5 2002" "10 5 4004" "76 2 2926"; do
  python tools/time_shape.py $s 400 --kernels 2>&1 | tail -2
  [ -n "$1" ] && python tools/time_shape.py $s 400 lib=$1 2>&1 | tail -1 | sed 's/^/  A: /'
done
python tools/time_shape.py 17 5 20349 10 --kernels 2>&1 | tail -2
[ -n "$1" ] && python tools/time_shape.py 17 5 20349 10 --kernels lib=$1 2>&1 | tail -2 | sed 's/^/  A: /'
python -c "from paper_2410_19844_b200 import build as b; b.build(experiments=True)" > /dev/null 2>&1
for s in "10 5 2002" "8 4 330"; do SOS_MID_TRACE=1 python tools/time_shape.py $s 3 --exp 2>&1 | grep -E "k_mid slowest" | tail -1; done
