# device timelines (steady state) at EP=1 and, with 4 GPUs, EP=4 — prologue diagnostics
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 2 --block-steps 200 --variant-steps 0 --no-twin"
CUDA_VISIBLE_DEVICES=0 timeout 300 python $B > gpurun_out/tl_ep1.log 2>&1
NG=$(nvidia-smi -L | wc -l)
[ $NG -ge 4 ] && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29571 $B --gpus 4 > gpurun_out/tl_ep4.log 2>&1
for f in gpurun_out/tl_ep1.log gpurun_out/tl_ep4.log; do
  [ -f $f ] && grep '^{' $f | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['n_gpus'], 'K', round(d['ms_per_step']*1e3,1), d['timeline_us'])"
done
