# checkpoint: full GPU suite, smoke, default bench line, config sweep
python -m pytest tests -q -m gpu > gpurun_out/r2_tests_c.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2_tests_c.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/r2_bench_c.json 2>gpurun_out/r2_bench_c.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/r2_bench_c.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['e2e']['value'],d['gpu_launches'],d['clocks'],d['cpu_baseline']['value'],d['cpu_baseline']['validation'])"
bash tools/sweep_configs.sh > gpurun_out/r2_sweep_c.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/r2_sweep_c.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'][:22], round(d['value'],2), round(d['ms_per_step'],4), d['gpu_launches'])
"
