"""Box topology + host<->device copy bandwidth per CPU placement: is the e2e
spread between runs a NUMA effect (pinned pages on the far socket)?
    python tools/microbench/numa_probe.py"""
import glob, json, os, subprocess, time
import torch

def bw(cpus):
    os.sched_setaffinity(0, cpus)
    n = 4096 * 2048 * 2
    hx = torch.empty(n, dtype=torch.uint8).pin_memory()
    ho = torch.empty(n, dtype=torch.uint8).pin_memory()
    dx = torch.empty(n, dtype=torch.uint8, device="cuda")
    do = torch.empty(n, dtype=torch.uint8, device="cuda")
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        steps = 100
        for _ in range(steps):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(up):
                    dx.copy_(hx, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(down):
                    ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
        res[mode] = round(n * steps * (2 if mode == "both" else 1) / (time.perf_counter() - t0) / 1e9, 1)
    return res

out = {"affinity": sorted(os.sched_getaffinity(0)), "cpu_count": os.cpu_count()}
out["nodes"] = {os.path.basename(p): open(p + "/cpulist").read().strip() for p in sorted(glob.glob("/sys/devices/system/node/node*"))}
try:
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
except Exception as e:
    out["topo"] = str(e)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
    out["nvml_gpu0_cpus"] = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
except Exception as e:
    out["nvml_gpu0_cpus"] = str(e)
allowed = sorted(os.sched_getaffinity(0))
torch.cuda.init()
res = {"all": bw(set(allowed))}
for node, lst in out["nodes"].items():
    cpus = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-"); cpus |= set(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    cpus &= set(allowed)
    if cpus:
        res[node] = bw(cpus)
out["copy_GBps"] = res
print(json.dumps(out))
