# short-K GEMMs with and without the bounded K-skew pacing (experiment build), k_mid trace
python -c "from paper_2410_19844_b200 import build as b; b.build(experiments=True)" > /dev/null 2>&1
for s in "8 4 330" "10 5 2002" "10 5 4004" "76 2 2926" "12 6 12376"; do
  st=400; [ "$s" = "12 6 12376" ] && st=20
  for ep in 8 0 32; do SOS_SKEW_EPOCH=$ep python tools/time_shape.py $s $st --exp --kernels 2>&1 | tail -2 | sed "s/^/ep=$ep /"; done
done
for s in "10 5 2002" "8 4 330"; do SOS_MID_TRACE=1 python tools/time_shape.py $s 3 --exp 2>&1 | grep -E "k_mid" | tail -2; done
