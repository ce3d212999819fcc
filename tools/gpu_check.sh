set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --steps 500 > gpurun_out/bench.log 2>&1; tail -c 3500 gpurun_out/bench.log
