# signalling ablation at P=2 and P=4 (group-size sweep + alpha-beta fits)
mkdir -p gpurun_out
rm -f gpurun_out/ablation.csv
for P in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port $((29700+P)) tools/ablate.py --steps 30 2>&1 | grep -v "^W\|OMP\|^\*" | tail -40
done
