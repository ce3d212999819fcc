# the round's bench lines: N = 1 (default invocation), 2 and 4 (torchrun), saved under gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29990+N)) bench.py --gpus $N > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err
done
for N in 1 2 4; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/final_n$N.json') if l.startswith('{')][-1])
print('N=$N', round(d['ms_per_step']*1e3,1), int(d['value']), 'e2e', int(d['e2e']['value']), 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'comm', None if not d['comm'] else round(d['comm']['exposed_frac'],3), 'variant', None if not d['per_tile_fence_variant'] else round(d['per_tile_fence_variant']['ms_per_step']*1e3,1))"; done
