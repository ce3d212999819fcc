# launch list + full ncu capture of the top kernels (run under gpurun, 1 GPU)
set -x
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_(gate|route|count|scatter|publish|plan|dispatch|gemm|combine)" -s 27 -c 45 \
  --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_gate|k_scatter|k_dispatch|k_combine" -s 15 -c 6 \
  -o gpurun_out/prof_r01 $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
