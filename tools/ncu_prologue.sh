# ncu launch durations of the short kernels before/after the fused kernel (EP=1 bench config)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --blocks 1 --block-steps 200 --variant-steps 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(gemm|route|perm|combine)" -s 20 -c 40 \
  --csv --log-file gpurun_out/prologue_launches.csv $B > gpurun_out/prologue_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/prologue_launches.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")))
for k, v in d.items():
    v.sort(); print(f"{k:40s} n={len(v):3d} median_us={v[len(v)//2]/1e3 if max(v)>1000 else v[len(v)//2]:.2f}")
PY
