# k_mid phase detail at configs 1 / 2 / 2b (experiment build)
python -c "from paper_2410_19844_b200 import build as b; b.build(experiments=True)" > /dev/null 2>&1
for s in "10 5 2002" "8 4 330" "10 5 4004"; do
  SOS_MID_TRACE=1 python tools/time_shape.py $s 4 --exp 2>&1 | grep -E "k_mid|steps/s" | tail -5
done
