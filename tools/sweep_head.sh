# EP=N: self-head scale x group size (same box)
cd $GRAFT_REPO_ROOT
N=${N:-4}
for hs in 1 2 0.5; do for gs in 0 -1; do
  PERSEUS_HEAD_SCALE=$hs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2981$N bench.py --gpus $N --steps 20 --warmup 5 --no-twin --variant-steps 0 --blocks 5 --block-steps 400 \
    --group-size $gs > gpurun_out/hs_${hs}_${gs}.log 2>&1
  grep '^{' gpurun_out/hs_${hs}_${gs}.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); c=d['comm']; pc=d['per_step_counters']
print('hs $hs gs $gs median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'mhz', d['clocks']['sm_mhz'],
      'wait_disp', round(pc['frac_wait_dispatch'],3), 'wait_g1', round(pc['frac_wait_g1'],3), 'mma_data', round(pc['frac_mma_data_wait'],3), 'fused', d['timeline_us'].get('fused'))"
done; done
