# final multi-GPU evidence: 4-GPU parity + device traces (one process per GPU), bench lines at EP=2/4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 \
  tests/mgpu_check.py > gpurun_out/r02_mgpu_check_ep4.log 2>&1
grep mgpu_check gpurun_out/r02_mgpu_check_ep4.log > gpurun_out/r02_mgpu_check_ep4.json
python -c "
import json; d=json.load(open('gpurun_out/r02_mgpu_check_ep4.json'))
print(d['mgpu_check'], [(r[0]['routing'], r[0]['protocol'], all(x['ok'] for x in r), r[0].get('rel_err')) for r in d['results']])
[print(t['protocol'], t['violations'], t['conservation'], t['dispatch']['fence_count'], t['dispatch']['flagged_signal_count']) for t in d['device_trace']]"
TAG=${TAG:-r02f} SKIP_NCCL=${SKIP_NCCL:-} bash tools/mgpu_bench.sh
