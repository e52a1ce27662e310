"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches and device
time per kernel, share of the total, and the largest launches."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}
by = collections.defaultdict(lambda: [0, 0.0])
launches = []
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0]
    ms = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    by[name][0] += 1
    by[name][1] += ms
    launches.append((int(d["ID"]), name, ms, d["Grid Size"]))
tot = sum(v[1] for v in by.values())
print(f"{len(launches)} launches, {tot:.3f} ms of device time (ncu, serialised, cold caches)")
print()
print("| kernel | launches | ms | share |")
print("|---|---|---|---|")
for k, (n, ms) in sorted(by.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
print()
print("largest launches (id, kernel, ms, grid):")
for b in sorted(launches, key=lambda x: -x[2])[:10]:
    print(f"  {b[0]:4d} {b[1]:24s} {b[2]:9.3f} {b[3]}")
