# descent floor under both readings of PAPER.md:218-219 (profiles/r2_descent_floor.md)
for c in c1_n8_2d8:6000 c2_n10_2d10:6000 c2b_n10_2d10_r4004:6000 c3_n12_2d12:2000 c4_n17_2d10:700; do
  w=${c%%:*}; s=${c##*:}
  timeout 400 python tools/descent_floor.py --config $w --steps $s --time-limit 240 > gpurun_out/r2_floor_$w.log 2>&1
  tail -1 gpurun_out/r2_floor_$w.log
done
