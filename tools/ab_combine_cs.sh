mkdir -p gpurun_out
# A/B of the combine kernel's streaming cache hints (PERSEUS_COMBINE_CS) on one box, alternated
for r in 1 2 3; do for v in 0 1; do
  PERSEUS_COMBINE_CS=$v timeout 300 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/cs_${v}_$r.json
  python -c "
import json; d=json.load(open('gpurun_out/cs_${v}_$r.json')); print('CS=$v run $r', round(d['ms_per_step']*1e3,2), 'combine', round(d['stage_ms']['combine']*1e3,2), 'clk', d['clocks']['sm_mhz'])"
done; done
PERSEUS_COMBINE_CS=1 timeout 600 python -m pytest tests/test_gpu_layer.py -x -q 2>&1 | tail -2
