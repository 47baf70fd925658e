"""Print the key counters of every launch in an ncu capture (run here, not on the box)."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(raw)))
hdr, units = rd[0], rd[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'lts__t_sector_hit_rate.pct', 'sm__inst_executed_pipe_lsu.sum']
for row in rd[2:]:
    m = dict(zip(hdr, row)); u = dict(zip(hdr, units))
    print(m.get('Kernel Name'), m.get('ID'))
    for k in keys:
        if k in m: print(f"   {k:75s} {m[k]:>16s} {u.get(k,'')}")
    st = {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]: float(v) for k, v in m.items()
          if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio') and 'not_issued' not in k and float(v) > 0.08}
    print("   stalls/issue:", dict(sorted(st.items(), key=lambda x: -x[1])))
    if len(sys.argv) > 2:
        for k, v in m.items():
            if sys.argv[2] in k: print("   ", k, v, u.get(k, ''))
