"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    k = r["Kernel Name"].split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n / steps:6.0f} launches {t / steps:9.1f} us/step  {t / n:7.1f} us/launch  {k}")
print(f"total {tot / steps:.1f} us/step")
