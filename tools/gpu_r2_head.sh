# round 2 re-entry: full GPU suite, smoke, default bench line and config sweep at HEAD
python -m pytest tests -q -m gpu -x --durations=12 > gpurun_out/h_tests.log 2>&1; echo tests_rc=$?; tail -16 gpurun_out/h_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/h_smoke.log
timeout 600 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo bench_rc=$?; tail -c 3000 gpurun_out/h_bench.json
bash tools/sweep_configs.sh > gpurun_out/h_sweep.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/h_sweep.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'][:22], round(d['value'],2), round(d['ms_per_step'],4), d['gpu_launches'])
"
