# round 2: split-step (k_mid + k_update_rows) vs fused step on short-K shapes, plus the affected GPU tests
python -m pytest tests -q -m gpu -x --durations=10 -k "variants or descend_matches or test_adam_and_gd or config0 or config1 or stop_rule or config2 or solve_host or smoke" > gpurun_out/t2.log 2>&1; echo rc=$?; tail -5 gpurun_out/t2.log
for cfg in "8 4 330" "10 5 2002" "10 5 4004" "5 3 35" "20 2 210" "30 2 465" "76 2 2926"; do
  for sp in 0 1; do timeout 120 python tools/time_shape.py $cfg 400 split=$sp --kernels; done
done 2>&1 | tee gpurun_out/t2_shapes.log
