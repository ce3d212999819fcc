"""Build profiles/<TAG>_qwen3_ep1_ncu_summary.json from the outputs of tools/gpu_profile.sh
(gpurun_out/launches_<TAG>.csv, prof_moe2_<TAG>.ncu-rep, bench_<TAG>.log), and
profiles/ncu_traffic.json (roofline.traffic in bench.py).  Runs here (ncu -i reads the
report without a GPU).
    python tools/ncu_summary.py TAG "what changed" """
import csv
import collections
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
FULL_METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "l1tex__m_l1tex2xbar_write_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
                "launch__block_size", "launch__cluster_dim_x", "launch__grid_size", "launch__registers_per_thread",
                "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__cycles_elapsed.avg.per_second",
                "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
                "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}


def launch_list(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        name = r["Kernel Name"].replace("perseus::", "").replace("void ", "").split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            per[name]["us"].append(v * SCALE.get(u, 1) / 1e-6 if u != "us" else v)
        elif r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[name][r["Metric Name"]].append(v * SCALE.get(u, 1))
    tot = sum(sum(d["us"]) for d in per.values())
    out = {}
    for name, d in sorted(per.items(), key=lambda kv: -sum(kv[1]["us"])):
        n = len(d["us"])
        out[name] = {"launches": n, "avg_us": round(sum(d["us"]) / n, 2),
                     "dram_read_MB": round(sum(d["dram__bytes_read.sum"]) / n / 1e6, 1),
                     "dram_write_MB": round(sum(d["dram__bytes_write.sum"]) / n / 1e6, 1),
                     "share": round(sum(d["us"]) / tot, 3)}
    return out


def full_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, v = r[0], r[1], r[2]
    m = {k: [x, u] for k, u, x in zip(h, units, v) if k in FULL_METRICS}
    rd = float(m["dram__bytes_read.sum"][0]) * SCALE[m["dram__bytes_read.sum"][1]]
    wr = float(m["dram__bytes_write.sum"][0]) * SCALE[m["dram__bytes_write.sum"][1]]
    return m, rd + wr


def main():
    tag, what = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    ll = launch_list(os.path.join(OUT, f"launches_{tag}.csv"))
    m, traffic = full_metrics(os.path.join(OUT, f"prof_moe2_{tag}.ncu-rep"))
    bench = [ln for ln in open(os.path.join(OUT, f"bench_{tag}.log")) if ln.startswith("{")]
    dur_us = float(m["gpu__time_duration.sum"][0]) * SCALE.get(m["gpu__time_duration.sum"][1], 1e-6) / 1e-6 \
        if m["gpu__time_duration.sum"][1] != "us" else float(m["gpu__time_duration.sum"][0])
    H, I, E, S, k = 2048, 768, 128, 4096, 8
    alg = E * 3.0 * H * I * 2 + 2.0 * S * H * 2  # expert weights + x + out
    summary = {
        "round": 2, "tag": tag, "what": what,
        "kernel": "k_moe2", "config": "qwen3 EP=1 S=4096 balanced",
        "duration_us": dur_us, "dram_bytes_per_launch": traffic,
        "dram_read_bytes": float(m["dram__bytes_read.sum"][0]) * SCALE[m["dram__bytes_read.sum"][1]],
        "dram_write_bytes": float(m["dram__bytes_write.sum"][0]) * SCALE[m["dram__bytes_write.sum"][1]],
        "algorithmic_bytes": alg, "traffic_ratio": traffic / alg,
        "dram_gbs": traffic / (dur_us * 1e-6) / 1e9,
        "sm_clock_hz": float(m["sm__cycles_elapsed.avg.per_second"][0]) * {"Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(
            m["sm__cycles_elapsed.avg.per_second"][1], 1.0),
        "tensor_pipe_pct": m["sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"][0],
        "tensor_mem_cycles_pct": m["sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0],
        "l2_hit_pct": m["lts__t_sector_hit_rate.pct"][0],
        "note": "ncu replays are cold-cache and serialised, at the clock ncu saw: compare the DRAM bytes and shares, "
                "not the absolute duration, with bench.py",
        "ncu_launch_list": {"cmd": "tools/gpu_profile.sh: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                                   "dram__bytes_write.sum --clock-control none (fused forward kernels, 3 forwards)",
                            "note": "cold-cache, serialised per-launch times: compare shares, not absolutes",
                            "per_kernel": ll},
        "ncu_full_k_moe2": {"cmd": "ncu --set full --clock-control none --import-source on -k regex:k_moe2 -s 3 -c 1 "
                                   "python bench.py (short run, see tools/gpu_profile.sh)",
                            "metrics": m},
        "bench_line": json.loads(bench[-1]) if bench else None,
    }
    path = os.path.join(ROOT, "profiles", f"{tag}_qwen3_ep1_ncu_summary.json")
    json.dump(summary, open(path, "w"), indent=1)
    print(path, {k: v["avg_us"] for k, v in ll.items()}, "traffic", traffic)


if __name__ == "__main__":
    main()
