# round 2: full GPU test suite + default bench line (+ short config sweep)
python -m pytest tests -q -m gpu -x --durations=12 > gpurun_out/r2_tests.log 2>&1; echo tests_rc=$?; tail -16 gpurun_out/r2_tests.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/r2_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['clocks'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
bash tools/sweep_configs.sh > gpurun_out/r2_sweep.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/r2_sweep.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'][:22], round(d['value'],2), round(d['ms_per_step'],4), d['gpu_launches'])
"
