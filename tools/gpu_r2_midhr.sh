python -m pytest tests -q -m gpu -x -k "variants or descend_matches or config1 or config2 or stop_rule or smoke or adam_and_gd or tiny or fuzz or split_config or solve_host" 2>&1 | tail -2
SOS_MID_TRACE=1 python tools/time_shape.py 10 5 2002 2 --exp 2>&1 | grep k_mid | tail -2
for s in "8 4 330" "10 5 2002" "10 5 4004" "20 2 210" "30 2 465" "76 2 2926"; do timeout 300 python tools/time_shape.py $s 400; done
