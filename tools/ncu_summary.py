"""Key metrics of each kernel in an ncu report (dev tool).  usage: ncu_summary.py rep [rep...]"""
import csv, io, subprocess, sys
KEYS = ['gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'sm__inst_executed.avg.per_cycle_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'l1tex__t_bytes.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']
STALL = 'smsp__average_warps_issue_stalled_'
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print("==", rep, v[h.index("Kernel Name")][:60])
        for k in KEYS:
            if k in h:
                print(f"  {k:70s} {v[h.index(k)]} {units[h.index(k)]}")
        st = [(k[len(STALL):-len('_per_issue_active.ratio')], float(v[i] or 0)) for i, k in enumerate(h)
              if k.startswith(STALL) and k.endswith('_per_issue_active.ratio') and v[i] not in ('', 'n/a')]
        st.sort(key=lambda t: -t[1])
        print("  stalls/issue:", ", ".join(f"{k} {x:.2f}" for k, x in st[:8]))
