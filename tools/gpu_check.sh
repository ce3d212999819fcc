set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_(gate|route|hist|perm|publish|plan|dispatch|gemm|combine)" -s 30 -c 50 \
  --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
