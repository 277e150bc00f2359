# descent evidence + MMA power microbenchmark (one gpurun call)
set -x
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mma_power tools/mma_power.cu -lcuda
for m in 0 1 2 3 4 5 6 7; do
  nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > gpurun_out/pw_$m.csv &
  SMI=$!
  sleep 0.5
  timeout 60 /tmp/mma_power $m 6 > gpurun_out/mma_$m.json
  kill $SMI
  sleep 2
done
timeout 900 python -m pytest tests -q -m gpu -k "stop_rule or descent" -s > gpurun_out/descent_tests.log 2>&1
for c in c3_n12_2d12 c4_n17_2d10; do
  timeout 300 python tools/descent.py --config $c --opt adam --lr 1e-3 --steps 1500 --log-every 50 > gpurun_out/descent_$c.log 2>&1
done
