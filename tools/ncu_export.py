"""Export the key metrics (+ hottest source lines) of ncu reports / metric CSVs
for profiles/ (dev tool).

usage: ncu_export.py full REP LIB KERNEL CAPTURE_NOTE OUT.json
       ncu_export.py metrics CSV OUT.json            (ncu --metrics --csv log)
"""
import csv, io, json, os, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum"]
STALL = "smsp__average_warps_issue_stalled_"


def full(rep, lib, kernel, note, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, res = rows[0], rows[1], []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90], "capture": note}
        for k in KEYS:
            if k in hdr:
                d[f"{k} [{units[hdr.index(k)]}]"] = r[hdr.index(k)]
        st = {h[len(STALL):].replace("_per_issue_active.ratio", ""): float(r[i] or 0)
              for i, h in enumerate(hdr) if h.startswith(STALL) and h.endswith("_per_issue_active.ratio")}
        d["stalls_per_issue_top"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])
        lines = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_lines.py"), rep, lib,
                                kernel, "25"], capture_output=True, text=True).stdout.splitlines()
        d["hot_source_lines"] = [ln.strip() for ln in lines if "% samp" in ln]
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)


def metrics(path, out):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i0]
    res = {}
    for r in rows[i0 + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        key = f"{d['Metric Name']} [{d['Metric Unit']}]"
        res.setdefault(name, {}).setdefault(key, d["Metric Value"])
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:7])
    else:
        metrics(sys.argv[2], sys.argv[3])
