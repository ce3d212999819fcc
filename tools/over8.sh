# 8 EP ranks on the 4 GPUs of this box (2 per GPU, grids capped to half the SMs, PDL off
# automatically since ranks share a device): 8-rank parity (tests/mgpu_check.py) and a
# functional run of bench.py's N=8 path (times are NOT 8-GPU NVLink timings)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PERSEUS_NUM_SMS=${PERSEUS_NUM_SMS:-74}
bash tools/mgpu8over.sh
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 8 --steps 10 --warmup 3 --blocks 2 --block-steps 200 --variant-steps 50 --no-cpu-baseline \
  > gpurun_out/bench_over8.log 2>&1
grep '^{' gpurun_out/bench_over8.log | tail -1 > gpurun_out/bench_over8.json
python -c "
import json; d=json.load(open('gpurun_out/bench_over8.json'))
print('N=8 over 4 GPUs: K us', round(d['ms_per_step']*1e3,1), 'tok/s', int(d['value']), 'gpu_launches', d['gpu_launches'],
      'dedup', (d.get('dedup_variant') or {}).get('wire_bytes_ratio_vs_this_run'), 'per-tile fences', d['per_tile_fence_variant']['fences_per_forward'])" \
  || tail -30 gpurun_out/bench_over8.log
