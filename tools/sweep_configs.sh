# bench.py on every BASELINE.json config (throughput table; config 4 is the headline).
# More timed steps for the small configs so the timed region is >= ~0.5 s.
for ws in c0_n4_2d6:4000 c1_n8_2d8:2000 c2_n10_2d10:1000 c2b_n10_2d10_r4004:400 c3_n12_2d12:60 c4_n17_2d10:20; do
  w=${ws%%:*}; s=${ws##*:}
  timeout 300 python bench.py --workload $w --steps $s --warmup 5 --no-e2e --no-cpu-baseline --kernel-timing separate 2>/dev/null
done
