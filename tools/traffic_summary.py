"""DRAM traffic of one full apply from an ncu per-launch CSV
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum):
per-kernel totals and the per-sweep DRAM bytes bench.py reports as
roofline.traffic (an IC apply runs two sweeps).  Run here, not on the box.

  python tools/traffic_summary.py <launches.csv[.gz]> <build hash> <out.json> [alg bytes per sweep]
"""
import collections
import csv
import gzip
import io
import json
import sys

path, build, out = sys.argv[1], sys.argv[2], sys.argv[3]
alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
raw = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = [l for l in raw.splitlines(True) if not l.startswith("==")]
rd = list(csv.reader(io.StringIO("".join(rows))))
hdr = rd[0]
ik, im, iv, iu = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rd[1:]:
    if len(r) <= iv:
        continue
    k = r[ik].split("(")[0]
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    agg[k][r[im]] += v
    if r[im] == "gpu__time_duration.sum":
        cnt[k] += 1
kern = {}
for k, m in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    kern[k] = {"launches": cnt[k], "time_ms": 1e3 * m["gpu__time_duration.sum"],
               "dram_read_gb": m["dram__bytes_read.sum"] / 1e9,
               "dram_write_gb": m["dram__bytes_write.sum"] / 1e9}
sweep = [k for k in kern if "sf_" in k]
tot_b = sum(1e9 * (kern[k]["dram_read_gb"] + kern[k]["dram_write_gb"]) for k in sweep)
tot_t = sum(kern[k]["time_ms"] for k in sweep)
res = {"source": path, "build": build, "sweeps_in_capture": 2,
       "dram_bytes_per_launch": tot_b / 2, "sweep_kernel_time_ms_per_sweep_under_ncu": tot_t / 2,
       "alg_bytes_per_sweep": alg, "traffic_over_algorithmic": (tot_b / 2 / alg) if alg else None,
       "kernels": kern}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: res[k] for k in res if k != "kernels"}, indent=1))
for k, v in kern.items():
    print(f"{k[:50]:50s} n={v['launches']:5d} {v['time_ms']:9.2f} ms  rd {v['dram_read_gb']:8.2f} GB  wr {v['dram_write_gb']:8.2f} GB")
