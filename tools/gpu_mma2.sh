nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/m2 tools/mma2_bench.cu
for n in 64 128 160 192 256; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/pw.csv & S=$!
  /tmp/m2 $n 0 1.5; kill $S; python3 -c "
import statistics; v=[l.split(',') for l in open('/tmp/pw.csv') if ',' in l]; v=[(float(a),float(b)) for a,b in v if float(b)>200]
print('   clk', statistics.median([x[0] for x in v]) if v else None, 'W', statistics.median([x[1] for x in v]) if v else None)"
done
for n in 160 256; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/pw.csv & S=$!
  /tmp/m2 $n 1 2; kill $S; python3 -c "
import statistics; v=[l.split(',') for l in open('/tmp/pw.csv') if ',' in l]; v=[(float(a),float(b)) for a,b in v if float(b)>200]
print('   clk', statistics.median([x[0] for x in v]) if v else None, 'W', statistics.median([x[1] for x in v]) if v else None)"
done
