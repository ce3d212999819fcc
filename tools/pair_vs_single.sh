# fused CTA-pair kernel vs the 1-CTA fused kernel (--no-pair) under skewed routing, N GPUs
N=${N:-1}
for R in ${ROUTES:-zipf:1.0 zipf:1.5}; do RT=${R%%:*}; SK=${R##*:}; for NP in "" "--no-pair"; do
  if [ $N = 1 ]; then CMD="python"; else CMD="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611"; fi
  timeout 400 $CMD bench.py --gpus $N --steps 300 --warmup 5 --no-cpu-baseline --variant-steps 0 --routing $RT --skew $SK $NP > gpurun_out/pvs.log 2>&1
  grep "^{" gpurun_out/pvs.log | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('N=$N $RT $SK $NP', round(d['ms_per_step']*1e3,1), d['cta_pairs'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/pvs.log
done; done
