# 8 EP ranks on the GPUs of this box (2 per GPU on 4 GPUs): each rank's persistent grids
# capped to half the SMs so two ranks' fused kernels are co-resident on one GPU.
export PERSEUS_NUM_SMS=${PERSEUS_NUM_SMS:-74}
N=${N:-8}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 tests/mgpu_check.py > gpurun_out/mgpu_over$N.log 2>&1
grep mgpu_check gpurun_out/mgpu_over$N.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['mgpu_check'], [(r['routing'], r['protocol'], r['ok']) for res in d['results'] for r in res[:1]]); [print(json.dumps({k: t[k] for k in ('protocol','violations','conservation')}), t['dispatch']['fence_count'], t['dispatch']['flagged_signal_count']) for t in d['device_trace']]" || tail -30 gpurun_out/mgpu_over$N.log
