# s8 MMA throughput / clock under the power cap vs operand digit width
for m in 4 8 9 7 4 8; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 200 > gpurun_out/smi_$m.csv &
  SP=$!
  ./tools/mma_power $m 6 160 > gpurun_out/mp_$m.json
  kill $SP
  python - "$m" <<'PY' >> gpurun_out/mp.log
import json, statistics, sys
m = sys.argv[1]
d = json.load(open(f"gpurun_out/mp_{m}.json"))
rows = [l.split(",") for l in open(f"gpurun_out/smi_{m}.csv") if l.strip()]
rows = [(float(a), float(b)) for a, b in rows if float(b) > 250]
print(m, d["tops"], d["mma_per_us_per_sm"], statistics.median(r[0] for r in rows) if rows else None, statistics.median(r[1] for r in rows) if rows else None)
PY
done
