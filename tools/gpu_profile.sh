# bench line + ncu launch list (+ DRAM bytes) + one full ncu capture of the fused kernel (EP=1)
set -x
TAG=${TAG:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; grep '^{' gpurun_out/bench_$TAG.log | tail -c 3000
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --blocks 3 --block-steps 200 --variant-steps 0"
timeout 300 $B > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(gate|route|perm|plan|gemm|combine|moe)" -s 18 -c 18 \
  --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_moe2" -s 3 -c 1 \
  -o gpurun_out/prof_moe2_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
