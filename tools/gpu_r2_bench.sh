# default bench line (config 4, cpu_baseline on the host cores) + the reference arm
python bench.py > gpurun_out/r2_bench_full.json 2> gpurun_out/r2_bench_full.err; echo bench_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo ref_rc=$?
tail -c 1500 gpurun_out/r2_ref.json
python -c "import json;d=json.loads(open('gpurun_out/r2_bench_full.json').read().strip().splitlines()[-1]);print(json.dumps(d['cpu_baseline'],indent=1));print(d['value'],d['roofline']['frac'],d['e2e'])"
