# k_moe2 in the tensor-bound regime at EP=1 (S tokens; 8192 => 512 rows/expert as at EP=2)
S=${S:-8192}
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tokens $S"
timeout 300 $B > gpurun_out/plain_t$S.log 2>&1; grep '^{' gpurun_out/plain_t$S.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('us', d['ms_per_step']*1e3, 'stages', d['stage_ms'], 'roof', d['roofline']['tensor'], d['roofline']['hbm'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_moe2" -s 3 -c 1 \
  -o gpurun_out/prof_moe2_t$S $B > gpurun_out/ncu_full_t$S.log 2>&1
tail -2 gpurun_out/ncu_full_t$S.log
