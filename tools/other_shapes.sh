# the other BASELINE shapes: Llama4-Scout and DeepSeek-V3 (EP = 1 and 4)
for CFG in llama4 dsv3; do for N in 1 4; do
  if [ $CFG = dsv3 ] && [ $N = 1 ]; then continue; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29850+N)) bench.py --gpus $N --config $CFG --steps 100 --warmup 5 --no-cpu-baseline --variant-steps 50 2>&1 | grep '^{' > gpurun_out/bench_${CFG}_n$N.json
  python -c "
import json; d=json.load(open('gpurun_out/bench_${CFG}_n$N.json'))
r=d['roofline']; lr=d['layer_roofline']
print('$CFG N=$N', round(d['ms_per_step']*1e3,1), 'us', int(d['value']), 'tok/s', r['bound'], round(r['frac'],3), 'tensor', round(r['tensor']['achieved_tflops']), 'TF', 'layer_frac', round(lr['frac'],3), 'comm', None if not d['comm'] else round(d['comm']['exposed_frac'],3))"
done; done
