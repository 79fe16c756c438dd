"""Attribute an ncu SASS source page to CUDA source lines (dev tool).

usage: python tools/ncu_lines.py report.ncu-rep lib.so kernel_substring [topN]
Joins `ncu --page source --print-source sass` (per-instruction samples and
executed counts) with `nvdisasm -g` line info of the same cubin.
"""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, check=True,
               capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
sass = []
for cf in cub:
    sass += subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cf)], capture_output=True,
                           text=True).stdout.splitlines()
addr2line = {}
infn = False
cur = None
for ln in sass:
    if ln.startswith("//-----") and ".text." in ln:
        infn = kname in ln
        continue
    if not infn:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# multiple kernels may be present; pick the block for kname
blocks, curb = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        curb = [ln]
        blocks.append(curb)
    elif curb is not None:
        curb.append(ln)
blk = next(b for b in blocks if kname in b[0])
rd = list(csv.reader(io.StringIO("\n".join(blk[1:]))))
hdr = rd[0]
ia = hdr.index("Address")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
agg = collections.defaultdict(lambda: [0, 0])
tot_s = tot_e = 0
base = None
for r in rd[1:]:
    try:
        a = int(r[ia], 16)
        if base is None:
            base = a
        a -= base
        s = float(r[isamp] or 0)
        e = float(r[iex] or 0)
    except (ValueError, IndexError):
        continue
    key = addr2line.get(a, ("?", 0))
    agg[key][0] += s
    agg[key][1] += e
    tot_s += s
    tot_e += e
src_cache = {}
def src(f, l):
    if f not in src_cache:
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2601_05765_b200", "csrc", f)
        src_cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
    L = src_cache[f]
    return L[l - 1].strip()[:90] if 0 < l <= len(L) else ""
print(f"total samples {tot_s:.0f}  instructions executed {tot_e:.3e}")
for (f, l), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*e/tot_e:5.1f}% inst  {f}:{l:<5d} {src(f, l)}")
