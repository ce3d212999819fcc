set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -c 2500 gpurun_out/bench.log
timeout 300 python bench.py --no-cpu-baseline --no-pair > gpurun_out/bench_nopair.log 2>&1; tail -c 2500 gpurun_out/bench_nopair.log
