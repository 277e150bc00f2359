# bench.py on every BASELINE.json config (throughput table; config 4 is the headline)
for w in c1_n8_2d8 c2_n10_2d10 c2b_n10_2d10_r4004 c3_n12_2d12 c4_n17_2d10; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null
done
