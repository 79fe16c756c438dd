"""Summarise an ncu --csv launch list (gpu__time_duration.sum) into a markdown table (dev tool).
usage: launch_table.py launches.csv"""
import csv, collections, io, sys
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
ik, iv, im, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
for r in rows[1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
tot = sum(v for _, v in agg.values())
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (c, v) in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"| {k} | {c} | {v:.3f} | {100 * v / tot:.1f}% |")
print(f"\ntotal {tot:.1f} ms over {sum(c for c, _ in agg.values())} launches")
