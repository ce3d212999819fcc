set -x
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain.log 2>&1; tail -c 600 gpurun_out/plain.log
timeout 300 $B --unfused > gpurun_out/plain_unfused.log 2>&1; tail -c 600 gpurun_out/plain_unfused.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none \
  -k regex:"k_(gate|route|hist|perm|publish|plan|dispatch|gemm|combine|moe)" -s 24 -c 24 \
  --csv --log-file gpurun_out/launches_fused.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_moe" -s 3 -c 1 \
  -o gpurun_out/prof_moe $B > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
