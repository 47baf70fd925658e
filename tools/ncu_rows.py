"""Key counters of every launch in an ncu --set full capture (run here, not on the box).

  python tools/ncu_rows.py <capture.ncu-rep> [out.json] ["source note"]
Prints one block per launch and, with out.json, writes the same numbers as a
list (the summaries kept under profiles/).  The FP64 tensor pipe is
sm__pipe_tensor_subpipe_dmma_cycles_active (sm__pipe_fp64_* does not see DMMA).
"""
import csv
import io
import json
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(raw)))
hdr, units = rd[0], rd[1]
keys = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "registers_per_thread": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dmma_pipe_active_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_inst_pct_of_peak": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
}
scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "second": 1e6}
out = []
for row in rd[2:]:
    m = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    d = {"kernel": m.get("Kernel Name"), "grid": m.get("Grid Size"), "block": m.get("Block Size")}
    for name, k in keys.items():
        if k in m:
            try:
                d[name] = float(m[k].replace(",", "")) * scale.get(u.get(k, ""), 1.0)
            except ValueError:
                pass
    st = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: round(float(v), 3)
          for k, v in m.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
          and "not_issued" not in k and float(v) > 0.08}
    d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1]))
    if "dram_read_bytes" in d and d.get("duration_us"):
        d["dram_gbs"] = (d["dram_read_bytes"] + d["dram_write_bytes"]) / d["duration_us"] / 1e3
    out.append(d)
    print(json.dumps(d, indent=1))
if len(sys.argv) > 2 and sys.argv[2].endswith(".json"):
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    json.dump({"source": note, "capture": sys.argv[1], "launches": out}, open(sys.argv[2], "w"), indent=1)
