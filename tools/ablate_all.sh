# signalling ablation: P=2 and P=4 on real GPUs (one process per GPU), P=8 as 8 ranks on one GPU
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ablation_r02.csv
for P in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2991$P \
    tools/ablate.py --out gpurun_out/ablation_r02.csv > gpurun_out/ablate_p$P.log 2>&1
  grep -E "^P=|alpha" gpurun_out/ablate_p$P.log
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/ablate_p8_onegpu.py > gpurun_out/ablate_p8.log 2>&1
grep -E "^P=|wrote|Error" gpurun_out/ablate_p8.log
