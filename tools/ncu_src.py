"""Summarise an ncu source-page CSV (SASS): top instructions by stall samples and shared-memory conflicts."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[col[k]] or 0)
    except: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print("total samples", tot)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(f(r, s) for r in data) for s in stalls}
print("stall mix:", {k: round(v / max(tot, 1), 3) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
print("--- top by samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(((f(r, s), s) for s in stalls), reverse=True)[:2]
    print(f"{f(r,'Warp Stall Sampling (All Samples)'):7.0f} {r[col['Address']]:>6} {r[col['Source']][:60]:60s} exec={f(r,'Instructions Executed'):.0f} conf={f(r,'L1 Conflicts Shared N-Way'):.0f} wfx={f(r,'L1 Wavefronts Shared Excessive'):.0f} {top}")
print("--- shared excessive wavefronts")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:8]:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"{r[col['Address']]:>6} {r[col['Source']][:70]:70s} wf={f(r,'L1 Wavefronts Shared'):.0f} ideal={f(r,'L1 Wavefronts Shared Ideal'):.0f}")
