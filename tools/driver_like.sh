# what the driver runs at round end (1 GPU)
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --impl reference > gpurun_out/ref_arm.json 2>&1; tail -c 600 gpurun_out/ref_arm.json
timeout 900 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','steps','warmup','gpu_launches')}, d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'], d['clocks'])"
