"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "nsecond"), 1e-3)
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{k[:58]:58s} n={n:5d} total={us:10.1f}us avg={us / n:9.2f}us share={us / tot:.3f}")
