"""Aggregate an ncu source page (--import-source, -lineinfo build) by code
region: the enclosing function of each CUDA source line of pf_cell.cuh, and
inside clip() its numbered steps (dev tool).

usage: python tools/ncu_regions.py report.ncu-rep lib.so kernel_substring
"""
import collections
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "..", "paper_2601_05765_b200", "csrc")


def region_map(fname):
    """line -> region name for one source file."""
    p = os.path.join(CSRC, fname)
    if not os.path.exists(p):
        return {}
    lines = open(p).read().splitlines()
    out, cur, step = {}, fname, None
    fn_re = re.compile(r"^(?:template <[^>]*>\s*)?(?:(?:PF_DEV|PF_NOINL|PF_PHASE|PF_HELPER|PF_WRED|__global__|__device__)[^(]*?"
                       r"|(?:int|void|double|bool|unsigned) )(\w+)\(")
    step_re = re.compile(r"^\s*// (\d[a-e]?)\. ")
    for i, ln in enumerate(lines, 1):
        m = fn_re.match(ln)
        if m:
            cur, step = m.group(1), None
        m = step_re.match(ln)
        if m and cur == "clip":
            step = m.group(1)
        out[i] = f"{cur}:{step}" if (cur == "clip" and step) else cur
    return out


def main():
    rep, so, kname = sys.argv[1:4]
    out = subprocess.run([sys.executable, os.path.join(HERE, "ncu_lines.py"), rep, so, kname, "100000"],
                         capture_output=True, text=True).stdout.splitlines()
    maps = {}
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for ln in out:
        m = re.match(r"\s*([\d.]+)% samp\s+([\d.]+)% inst\s+(\S+):(\d+)", ln)
        if not m:
            continue
        s, e, f, l = float(m.group(1)), float(m.group(2)), m.group(3), int(m.group(4))
        if f not in maps:
            maps[f] = region_map(f)
        reg = maps[f].get(l, f)
        agg[reg][0] += s
        agg[reg][1] += e
    print(out[0] if out else "")
    print(f"{'region':40s} {'%samples':>9s} {'%inst':>7s}")
    for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if s >= 0.2 or e >= 0.2:
            print(f"{k:40s} {s:9.1f} {e:7.1f}")


if __name__ == "__main__":
    main()
