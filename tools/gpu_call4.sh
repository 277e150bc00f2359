set -x
c=c3_n12_2d12
timeout 200 python tools/descent.py --config $c --opt adam --lr 1e-3 --decay 0.5 --steps 3000 --log-every 25 > gpurun_out/d4_a.log 2>&1
timeout 200 python tools/descent.py --config $c --opt adam --lr 3e-4 --steps 3000 --log-every 50 > gpurun_out/d4_b.log 2>&1
timeout 200 python tools/descent.py --config $c --opt adam --lr 5e-4 --decay 0.5 --steps 3000 --log-every 25 > gpurun_out/d4_c.log 2>&1
timeout 200 python tools/descent.py --config c4_n17_2d10 --opt adam --lr 1e-3 --decay 0.5 --steps 1000 --log-every 25 > gpurun_out/d4_d.log 2>&1
