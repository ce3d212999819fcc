# same-box alternating A/B of environment switches at N GPUs (one process per GPU):
#   N=4 SETS="A=0 A=1" REPS=2 bash tools/sweep_env_mgpu.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${N:-4}
B="bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline --blocks 5 --block-steps 300 --variant-steps 0 --no-twin $BENCH_ARGS"
for rep in $(seq ${REPS:-2}); do for s in $SETS; do
  tag=$(echo $s | tr ',=' '__')
  env $(echo $s | tr ',' ' ') timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) $B > gpurun_out/swm_$tag.log 2>&1
  grep '^{' gpurun_out/swm_$tag.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('$s N=$N median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'min', round(d['timing_blocks']['min_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'mhz', d['clocks']['sm_mhz'], 'fused', d['timeline_us'].get('fused'))" || tail -5 gpurun_out/swm_$tag.log
done; done
