"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per launch)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]; c = {h: j for j, h in enumerate(hdr)}
per = defaultdict(dict)
order = []
for r in rows[i + 1:]:
    if len(r) < len(hdr): continue
    try: v = float(r[c["Metric Value"]].replace(",", ""))
    except ValueError: continue
    key = (r[c["ID"]], r[c["Kernel Name"]])
    if key not in per: order.append(key)
    per[key][r[c["Metric Name"]]] = (v, r[c["Metric Unit"]])
agg = defaultdict(lambda: [0, 0.0, 0.0])
lines = []
for key in order:
    d = per[key]; name = key[1].split("(")[0].replace("void ", "").replace("tsqr::", "")
    t = d.get("gpu__time_duration.sum", (0, ""))
    tms = t[0] / 1e6 if t[1] == "ns" else (t[0] / 1e3 if t[1] == "us" else t[0])
    byt = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if m in d:
            v, u = d[m]; byt += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    agg[name][0] += 1; agg[name][1] += tms; agg[name][2] += byt
    lines.append((key[0], name, tms, byt))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':34s} {'n':>5s} {'ms':>9s} {'share':>6s} {'GB':>8s} {'GB/s':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {v[0]:5d} {v[1]:9.3f} {v[1]/tot:6.3f} {v[2]/1e9:8.2f} {v[2]/1e6/max(v[1],1e-9):8.0f}")
print("total ms", round(tot, 3))
if "-v" in sys.argv:
    for l in lines: print(f"{l[0]:>5s} {l[1]:34s} {l[2]:9.3f} ms {l[3]/1e9:7.2f} GB")
