for rep in 1 2 3; do
for r in 20349 20320; do timeout 300 python tools/time_shape.py 17 5 $r 20 >> gpurun_out/ts.log 2>&1; done
done
