# the other BASELINE shapes: Llama4-Scout and DeepSeek-V3 (EP = 1 and 4)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02}
for CFG in llama4 dsv3; do for N in 1 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29850+N)) \
    bench.py --gpus $N --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --variant-steps 50 --blocks 3 --block-steps 200 \
    2>&1 | grep '^{' > gpurun_out/${TAG}_bench_${CFG}_n$N.json
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench_${CFG}_n$N.json'))
r=d['roofline']; lr=d['layer_roofline']; c=d['comm']
print('$CFG N=$N', round(d['ms_per_step']*1e3,1), 'us', 'median', round(d['timing_blocks']['median_ms']*1e3,1), int(d['value']), 'tok/s', r['bound'], 'frac', round(r['frac'],3), 'tl', r.get('device_timeline',{}).get('frac_burst'), 'tensor', round(r['tensor']['achieved_tflops']), 'TF', 'pairs', d['cta_pairs'], 'layer_frac', round(lr['frac'],3), 'exposed', None if not c or not c.get('exposed') else round(c['exposed']['frac'],3), 'mhz', d['clocks']['sm_mhz'])"
done; done
