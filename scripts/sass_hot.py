"""Top stalled SASS instructions of one kernel from `ncu -i rep --page source --csv --print-source sass`.
    python scripts/sass_hot.py sass.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
def num(x):
    try:
        float(x or 0)
        return True
    except ValueError:
        return False
# first kernel block only (a capture of several launches repeats the header)
data = []
for r in rows[2:]:
    if len(r) > 1 and r[0] == "Kernel Name":
        break
    if len(r) > 2 and num(r[2]):
        data.append(r)
iS = h.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iS] or 0) for r in data)
print("total samples", tot)
agg = {}
for r in data:
    for i in stalls:
        agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
print("by reason:", sorted(((round(v / tot, 3), k) for k, v in agg.items() if v), reverse=True)[:10])
data.sort(key=lambda r: -float(r[iS] or 0))
for r in data[:top]:
    rs = sorted(((float(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:3]
    print(f"{float(r[iS] or 0) / tot:6.3f} {r[0]:>6} {r[1][:70]:70s} {rs}")
