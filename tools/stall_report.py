"""Summarise an ncu source page (SASS) into stall reasons + top instructions.
usage: python tools/stall_report.py rep.ncu-rep [top]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi]
iA, iS, iE, iW = (h.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"))
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[iA], 16), r[iS], int(r[iE] or 0), int(r[iW] or 0), r))
    except (ValueError, IndexError):
        continue
base = data[0][0]
tot = sum(d[3] for d in data)
agg = {}
for d in data:
    for i in cols:
        try: agg[h[i]] = agg.get(h[i], 0) + int(d[4][i] or 0)
        except ValueError: pass
print("samples", tot, "code bytes", hex(data[-1][0] - base))
print(", ".join(f"{k[6:]} {v/tot:.0%}" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
for d in sorted(data, key=lambda d: -d[3])[:top]:
    st = {h[i][6:]: d[4][i] for i in cols if d[4][i] not in ("0", "")}
    print(f"{d[0]-base:6x} exec={d[2]:>8} samples={d[3]:>5} {d[1][:48]:48s} {st}")
