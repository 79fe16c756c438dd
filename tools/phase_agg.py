"""Aggregate tools/ncu_lines.py output into line ranges (dev tool).
usage: phase_agg.py lines.txt name:a-b [name:a-b ...]"""
import re, sys
R = []
for spec in sys.argv[2:]:
    n, rng = spec.split(":")
    a, b = rng.split("-")
    R.append((n, int(a), int(b)))
agg = {k: [0.0, 0.0] for k, _, _ in R}
other = [0.0, 0.0]
for ln in open(sys.argv[1]):
    m = re.match(r"\s*([\d.]+)% samp\s+([\d.]+)% inst\s+(\S+):(\d+)", ln)
    if not m:
        continue
    s, i, f, l = float(m.group(1)), float(m.group(2)), m.group(3), int(m.group(4))
    for k, a, b in R:
        if f == "pf_cell.cuh" and a <= l <= b:
            agg[k][0] += s; agg[k][1] += i
            break
    else:
        other[0] += s; other[1] += i
for k, (s, i) in sorted(agg.items(), key=lambda t: -t[1][0]):
    print(f"{k:14s} samp {s:5.1f}%  inst {i:5.1f}%")
print(f"{'other':14s} samp {other[0]:5.1f}%  inst {other[1]:5.1f}%")
