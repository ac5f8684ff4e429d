"""Summarise a round's ncu evidence into profiles/<tag>/: the launch list (per-kernel device
time and DRAM bytes, cold-cache and serialised), the per-kernel `--set full` details exports,
and profiles/ncu_traffic_r01.json (DRAM bytes per launch per kernel class, read by bench.py
for roofline.traffic).

usage: python tools/profile_summary.py <tag> [algo_config]
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
config = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", tag)
os.makedirs(dst, exist_ok=True)

CLASS = {"k_update": "update", "k_update_pp": "update", "k_proj": "proj", "k_trmm": "trmm", "k_chol_inv": "chol",
         "k_chol_inv_blocked": "chol", "k_reduce": "reduce", "k_reduce_allreduce": "allreduce",
         "k_cluster_factor": "cluster", "k_chol_prep": "chol", "k_chol_diag": "chol", "k_chol_row": "chol",
         "k_chol_trail": "chol", "k_adapt_decide": "small", "k_adapt_resume": "small"}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)


# ---- launch list
rows = list(csv.reader(open(os.path.join(src, f"launches_{tag}.csv"))))
i0 = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i0]
c = {h: j for j, h in enumerate(hdr)}
per = {}
order = []
for r in rows[i0 + 1:]:
    if len(r) < len(hdr):
        continue
    try:
        v = float(r[c["Metric Value"]].replace(",", ""))
    except ValueError:
        continue
    key = (int(r[c["ID"]]), r[c["Kernel Name"]].split("(")[0].replace("void ", "").replace("tsqr::", ""))
    if key not in per:
        per[key] = {}
        order.append(key)
    per[key][r[c["Metric Name"]]] = v * unit_scale(r[c["Metric Unit"]])
with open(os.path.join(dst, "ncu_launches.csv"), "w") as f:
    f.write("id,kernel,ms,dram_read_bytes,dram_write_bytes\n")
    for key in order:
        d = per[key]
        f.write(f"{key[0]},{key[1]},{d.get('gpu__time_duration.sum', 0):.6f},"
                f"{d.get('dram__bytes_read.sum', 0):.0f},{d.get('dram__bytes_write.sum', 0):.0f}\n")
agg = defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
for key in order:
    name = key[1].split("<")[0]
    cls = CLASS.get(name, "small")
    d = per[key]
    agg[cls]["launches"] += 1
    agg[cls]["ms"] += d.get("gpu__time_duration.sum", 0.0)
    agg[cls]["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(v["ms"] for v in agg.values())
summary = {"tag": tag, "config": config, "total_ms": tot,
           "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   "--clock-control none -k regex:^k_ over bench.py --steps 1 --warmup 1 (2 factorisations): "
                   "cold-cache, serialised launches -- compare shares, not absolutes",
           "classes": {k: dict(v, share=v["ms"] / tot, dram_bytes_per_launch=v["dram_bytes"] / v["launches"])
                       for k, v in agg.items()}}
json.dump(summary, open(os.path.join(dst, "ncu_launch_summary.json"), "w"), indent=1)
traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic_r01.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
traffic[config] = {k: v["dram_bytes"] / v["launches"] for k, v in agg.items()}
json.dump(traffic, open(traffic_path, "w"), indent=1)

# ---- full captures -> details csv + a few headline metrics
heads = {}
for fn in sorted(os.listdir(src)):
    if fn.startswith(f"prof_{tag}_") and fn.endswith(".ncu-rep"):
        k = fn[len(f"prof_{tag}_"):-len(".ncu-rep")]
        rep = os.path.join(src, fn)
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        open(os.path.join(dst, f"ncu_{k}_details.csv"), "w").write(det)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        if len(rr) >= 3:
            h, u = rr[0], rr[1]
            want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
                    "launch__grid_size", "launch__block_size"]
            nm = h.index("Kernel Name") if "Kernel Name" in h else None
            heads[k] = [dict({"kernel": r[nm] if nm is not None else ""},
                             **{w: f"{r[h.index(w)]} {u[h.index(w)]}" for w in want if w in h}) for r in rr[2:]]
json.dump(heads, open(os.path.join(dst, "ncu_full_headlines.json"), "w"), indent=1)
print(json.dumps(summary["classes"], indent=1))
print(json.dumps(heads, indent=1)[:3000])
