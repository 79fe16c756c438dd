"""CPU Newton restatement (oracle/newton_ref.py over the reference-faithful
oracle) on a full benchmark configuration, as a committed fixture for the
device-vs-restatement Newton parity tests (tests/test_gpu_newton_sizes.py).

Writes tests/golden/newton_<cfg>.npz: psi (float32; the tests compare to
1e-6 relative), iteration / evaluation / CG counts, worst-error history, the
per-iteration CG counts, and the wall time on this host.

usage: python tools/newton_cpu_fixtures.py C2 [C3 C5] [--threads N]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    from oracle import newton_ref
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre, scenes

    O.set_threads(a.threads)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    for cfg in a.configs:
        sc = scenes.make(cfg)
        t0 = time.perf_counter()
        psi, st = newton_ref.newton_solve(sc.pts, sc.nu, dpk.args(), dpk.tol, dom.diagonal())
        dt = time.perf_counter() - t0
        keep = {k: st[k] for k in ("iterations", "evaluations", "cg_iterations", "damping_halvings",
                                   "init_doublings", "status", "worst_initial", "worst_final")}
        keep.update(cg_per_iter=[int(x) for x in st["cg_per_iter"]],
                    worst_history=[float(x) for x in st["worst_history"]],
                    seconds=dt, threads=O.num_threads(), n=sc.n, cpu=os.uname().machine)
        np.savez_compressed(os.path.join(a.out, f"newton_{cfg}.npz"), psi=psi.astype(np.float32),
                            meta=json.dumps(keep))
        print(cfg, json.dumps(keep), flush=True)


if __name__ == "__main__":
    main()
