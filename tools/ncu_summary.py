"""Summaries of the ncu captures kept under profiles/ (run here, not on the box).

  python tools/ncu_summary.py launches <launches.csv> <out.txt> "<command line>"
      per-kernel launch counts, total / per-launch time and share of the step
      (cold-cache, serialised launch list: shares are what must agree with the
      live timing, not absolute times)
  python tools/ncu_summary.py full <capture.ncu-rep> <out.json> "<source note>"
      the numbers DESIGN.md and bench.py cite for the sweep kernel: DRAM
      traffic per launch, duration under ncu, registers, shared memory,
      pipe utilisation and the warp-stall breakdown
"""
import csv
import io
import json
import subprocess
import sys


def launches(path, out, cmd):
    rows = [l for l in open(path) if not l.startswith("==")]
    rd = list(csv.reader(io.StringIO("".join(rows))))
    hdr = rd[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = {}
    for r in rd[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        k = r[ik][:60]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r[iv].replace(",", "")) / 1e3)
    tot = sum(t for _, t in agg.values())
    with open(out, "w") as f:
        f.write(cmd + "\n")
        f.write("cold-cache serialised launch times (ncu --metrics gpu__time_duration.sum --clock-control none)\n")
        f.write(f"{'kernel':60s} {'launches':>9s} {'total us':>12s} {'share':>7s} {'us/launch':>10s}\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k:60s} {n:9d} {t:12.1f} {100 * t / tot:6.1f}% {t / n:10.1f}\n")
    print(open(out).read())


def full(rep, out, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rd[0], rd[1], rd[2]
    m = dict(zip(hdr, vals))
    un = dict(zip(hdr, units))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
             "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
             "Kbyte/block": 1e3, "byte/block": 1.0}

    def g(k):  # SI base units (bytes, seconds) where ncu reports a unit
        try:
            return float(m[k].replace(",", "")) * scale.get(un.get(k, ""), 1.0)
        except (KeyError, ValueError):
            return None

    stalls = {}
    for k, v in m.items():
        pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
        if k.startswith(pre) and k.endswith(suf) and "not_issued" not in k:
            name = k[len(pre):-len(suf)]
            try:
                x = float(v)
            except ValueError:
                continue
            if x > 0.02:
                stalls[name] = round(x, 4)
    rd_b, wr_b = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    res = {
        "kernel": m.get("Kernel Name"),
        "source": note,
        "dram_bytes_per_launch": (rd_b or 0) + (wr_b or 0),
        "dram_read_bytes": rd_b,
        "dram_write_bytes": wr_b,
        "duration_ms_under_ncu": (g("gpu__time_duration.sum") or 0) * 1e3,
        "registers_per_thread": g("launch__registers_per_thread"),
        "dynamic_smem_per_block_kb": (g("launch__shared_mem_per_block_dynamic") or 0) / 1e3,
        "inst_executed": g("smsp__inst_executed.sum"),
        "sm_throughput_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "stall_ratios_per_issue": dict(sorted(stalls.items())),
    }
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4])
